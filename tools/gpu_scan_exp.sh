timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for S in 1 0; do TJ_SCAN3=$S python bench.py --no-cpu-baseline --no-e2e --steps 8 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('SCAN3=$S', 'ms/step', round(d['ms_per_step'],3), 'p50', round(d['p50_tick_ms'],3), d['stage_ms'])"; done
