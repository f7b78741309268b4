#!/bin/bash
# Development aid (runs on the GPU box): rebuild the library with tuning macros and
# run the order sweep for the given orders. usage: tools/tune_orders.sh "orders" "name|EXTRA flags" ...
orders="$1"; shift
for spec in "$@"; do
  name="${spec%%|*}"; extra="${spec#*|}"
  make -C paper_2605_16684_b200/csrc -j16 EXTRA="$extra" > /tmp/tune_build.log 2>&1 || { echo "$name: build failed"; tail -3 /tmp/tune_build.log; continue; }
  echo "== $name"
  python tools/sweep_probe.py $orders 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(' N=%d %s: stage %.3f GDOF/s (%.3f ms/launch) | split %.3f (K1 %.3f K2 %.3f)' % (d['order'], d['precision'], d['stage']['gdof_s'], d['stage']['vol_ms'], d['split']['gdof_s'], d['split']['vol_ms'], d['split']['surf_ms']))
"
done
make -C paper_2605_16684_b200/csrc -j16 > /dev/null 2>&1
