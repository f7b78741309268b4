"""Attributes warp-stall samples and issued instructions of one kernel to the
code regions between block barriers (phase A / x sweep / y sweep / ...), from
`ncu --page source --csv` of a report captured with --import-source on."""
import csv
import subprocess
import sys
import io

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# the page holds one block per kernel: a "Kernel Name" line, a header line, rows
want = sys.argv[2] if len(sys.argv) > 2 else None
blocks, cur_name = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur_name = r[1]
        blocks.append([cur_name, None, []])
    elif blocks and blocks[-1][1] is None:
        blocks[-1][1] = r
    elif blocks:
        blocks[-1][2].append(r)
blk = next((b for b in blocks if want is None or want in b[0]), blocks[0])
print("kernel:", blk[0][:100])
hdr = blk[1]
idx = {h: i for i, h in enumerate(hdr)}
data = blk[2]
seg, segs = [], []
for r in data:
    if len(r) < len(hdr):
        continue
    seg.append(r)
    if "BAR.SYNC" in r[idx["Source"]]:
        segs.append(seg)
        seg = []
segs.append(seg)
tot_s = sum(int(r[idx["# Samples"]]) for r in data if len(r) >= len(hdr))
tot_i = sum(int(r[idx["Instructions Executed"]]) for r in data if len(r) >= len(hdr))
print(f"total samples {tot_s}, warp instructions {tot_i}")
stall_cols = [h for h in hdr if h.startswith("stall_")] or [h for h in hdr if "Stall" in h]
for k, sg in enumerate(segs):
    s = sum(int(r[idx["# Samples"]]) for r in sg)
    i = sum(int(r[idx["Instructions Executed"]]) for r in sg)
    dp = sum(int(r[idx["Instructions Executed"]]) for r in sg
             if any(op in r[idx["Source"]] for op in ("DFMA", "DMUL", "DADD", "DSETP")))
    print(f"segment {k}: static {len(sg):5d}  samples {s:7d} ({s / tot_s:5.1%})  warp-instr {i:10d} ({i / tot_i:5.1%})  "
          f"DP share {dp / max(i, 1):5.1%}  samples/instr {s / max(i, 1) * 1e3:7.2f}e-3")
    top = sorted(sg, key=lambda r: -int(r[idx["# Samples"]]))[:6]
    for r in top:
        print(f"      {int(r[idx['# Samples']]):6d}  {r[idx['Source']].strip()[:70]}")
