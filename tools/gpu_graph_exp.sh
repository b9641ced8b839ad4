for G in 0 1; do TJ_NO_GRAPH=$G python bench.py --no-cpu-baseline --no-e2e --steps 8 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('NO_GRAPH=$G', 'ms/step', round(d['ms_per_step'],3), 'p50', round(d['p50_tick_ms'],3), 'dev_total', round(d['stage_ms']['total'],3), d['stage_ms'])"; done
