#!/bin/bash
# Development aid (runs on the GPU box): A/B timing of two builds of the library in one run,
# alternating, so that box-to-box and minute-to-minute differences (power cap) cancel.
# usage: tools/ab_probe.sh <libA.so> <libB.so> [perf_probe args]
A="$1"; B="$2"; shift 2
for rep in 1 2 3; do
  for lib in "$A" "$B"; do
    ESDG_B200_LIB="$lib" python tools/perf_probe.py --reps 3 "$@" | python -c "
import json,sys
d=json.load(sys.stdin)
print('$lib'[-40:], '| K1 %.3f ms | K2 %.3f | fused %.3f | stage %.3f' % (d['split']['volume_ms'], d['split']['surface_ms'], d['fused']['volume_ms'], d['stage']['volume_ms']))
"
  done
done
