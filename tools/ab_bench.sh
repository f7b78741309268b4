#!/bin/bash
# Development aid (runs on the GPU box): bench.py with two builds of the library, alternating.
# usage: tools/ab_bench.sh <libA.so> <libB.so> [bench.py args]
A="$1"; B="$2"; shift 2
for rep in 1 2 3; do
  for lib in "$A" "$B"; do
    ESDG_B200_LIB="$lib" python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('$lib'[-40:], '| %.3f ms/step | stage kernel %.3f ms | %.4g %s | clocks %s %s' % (d['ms_per_step'], d['roofline']['ms_per_launch'], d['value'], d['unit'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons')))
"
  done
done
