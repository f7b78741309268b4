"""Per-instruction stall breakdown of one kernel from `ncu --page source --csv`
(development aid). Usage: ncu_stalls.py source.csv [first_addr_offset last_addr_offset]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) >= len(hdr)]
base = int(data[0][0], 16)
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 60
cols = ["stall_wait", "stall_no_inst", "stall_short_sb", "stall_long_sb", "stall_math",
        "stall_not_selected", "stall_selected", "stall_barrier", "stall_mio", "stall_dispatch",
        "stall_branch_resolving", "stall_lg"]
tot = {c: 0 for c in cols}
ninst = 0
for r in data:
    off = int(r[0], 16) - base
    if off < lo or off > hi:
        continue
    ninst += int(r[idx["Instructions Executed"]])
    for c in cols:
        tot[c] += int(r[idx[c]])
s = sum(tot.values())
print(f"range {lo:#x}-{hi:#x}: warp-instr {ninst}, samples {s}")
for c in sorted(cols, key=lambda c: -tot[c]):
    print(f"  {c:24s} {tot[c]:8d}  {tot[c] / max(s, 1):6.1%}")
if "--list" in sys.argv:
    for r in data:
        off = int(r[0], 16) - base
        if off < lo or off > hi:
            continue
        st = " ".join(f"{c[6:9]}={r[idx[c]]}" for c in cols[:7] if int(r[idx[c]]) > 0)
        print(f"{off:5x} {r[idx['Source']].strip()[:52]:52s} n={r[idx['# Samples']]:>5s} {st}")
