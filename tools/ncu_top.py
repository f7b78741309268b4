"""Hottest instructions of one kernel from `ncu --page source --csv`
(development aid). Usage: ncu_top.py source.csv [count]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) >= len(hdr)]
base = int(data[0][0], 16)
tot = sum(int(r[idx['# Samples']]) for r in data)
print('total samples', tot)
top = sorted(data, key=lambda r: -int(r[idx['# Samples']]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]
cols = ["stall_long_sb", "stall_barrier", "stall_wait", "stall_short_sb", "stall_math", "stall_mio", "stall_lg", "stall_no_inst"]
for r in sorted(top, key=lambda r: int(r[0], 16)):
    off = int(r[0], 16) - base
    st = " ".join(f"{c[6:]}={r[idx[c]]}" for c in cols if int(r[idx[c]]) > 200)
    print(f"{off:6x} {r[idx['Source']].strip()[:60]:60s} n={r[idx['# Samples']]:>6s} {st}")
