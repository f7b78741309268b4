#!/bin/bash
cd paper_2605_16684_b200/csrc
for spec in "$@"; do
  name="${spec%%|*}"; extra="${spec#*|}"
  rm -f build/inst_nq5.o
  make -j8 EXTRA="$extra" > /dev/null 2>&1 || { echo "$name: build failed"; continue; }
  echo "== $name"
  (cd ../.. && python tools/perf_probe.py --reps 1 $PROBE_ARGS 2>&1 | grep "phase clocks" | sort | uniq -c | sort -rn | head -12)
done
rm -f build/inst_nq5.o; make -j8 > /dev/null 2>&1
