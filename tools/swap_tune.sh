for cfg in "8 32" "16 32" "4 32" "8 16" "8 64" "8 128" "16 64"; do set -- $cfg; ESDG_B200_SWAP_RUNS=$1 ESDG_B200_SWAP_PIECE_MB=$2 python bench.py --no-cpu-baseline --steps 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('runs $1 piece $2 MiB: e2e %.4g (sequential %.4g)' % (d['e2e']['value'], d['e2e']['sequential_value']))"; done
