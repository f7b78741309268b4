"""FP64 pipe cycles a kernel really needs on sm_100a, from `ncu --page source
--csv`: an FP64 instruction occupies the pipe for 2 cycles per warp, 3 when it
reads three distinct vector registers (tools/ubench/fp64_operands_ubench.cu);
operands flagged .reuse are served by the operand cache."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) >= len(hdr)]
n2 = n3 = n3r = 0
for r in data:
    s = re.sub(r"^@!?U?P\d\s+", "", r[idx["Source"]].strip())
    m = re.match(r"(DFMA|DMUL|DADD|DSETP)\S*\s+(.*)", s)
    if not m:
        continue
    ops = [o.strip() for o in m.group(2).split(",")]
    srcs = ops[1:] if m.group(1) != "DSETP" else ops[2:]
    regs, reused = set(), 0
    for o in srcs:
        mm = re.match(r"[-|]*\s*(R\d+)(\.reuse)?", o)
        if mm and mm.group(1) != "RZ":
            if mm.group(2):
                reused += 1
            regs.add(mm.group(1))
    ex = int(r[idx["Instructions Executed"]])
    if len(regs) >= 3:
        n3 += ex
        if reused:
            n3r += ex
    else:
        n2 += ex
tot = n2 + n3
print(f"FP64 warp-instructions {tot}: {n3} ({n3 / tot:.1%}) read 3 distinct vector registers "
      f"({n3r} of them carry a .reuse flag)")
print(f"pipe cycles per instruction: {(2 * n2 + 3 * n3) / tot:.3f} (2.000 nominal)")
