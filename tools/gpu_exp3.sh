for L in ${LIBS}; do echo "LIB=$L"; TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('VALUE',d['value'],d['stage_ms']['build'], d['stage_ms']['total'])"; done
