for D in ${DBGS:-0 4}; do echo "DBG=$D"; TJ_DEBUG=$D python bench.py --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('VALUE',d['value'],d['stage_ms'])"; done
