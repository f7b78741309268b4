#!/bin/bash
# Development aid (runs on the GPU box): rebuild inst_nq5 with tuning macros and time the FP32 kernels.
cd paper_2605_16684_b200/csrc
for spec in "$@"; do
  name="${spec%%|*}"; extra="${spec#*|}"
  rm -f build/inst_nq5.o
  make -j8 EXTRA="$extra" > /tmp/b.log 2>&1 || { echo "$name: build failed"; tail -3 /tmp/b.log; continue; }
  regs=$(cuobjdump -res-usage build/inst_nq5.o 2>&1 | grep -A1 "rhs_kernelIfLi5" | grep -o "REG:[0-9]* STACK:[0-9]*" | tr '\n' ' ')
  (cd ../.. && python tools/perf_probe.py --precision f32 --reps 2 2>&1 | python -c "
import json,sys
d=json.load(sys.stdin)
print('$name', '| K1 %.3f ms | K2 %.3f | fused %.3f | stage %.3f' % (d['split']['volume_ms'], d['split']['surface_ms'], d['fused']['volume_ms'], d['stage']['volume_ms']), '| $regs')
")
done
rm -f build/inst_nq5.o; make -j8 > /dev/null 2>&1
