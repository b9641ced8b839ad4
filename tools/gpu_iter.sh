# iteration: parity tests, one bench line, ncu of chosen kernels
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; echo bench=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]);print('VALUE',d['value'],'ms',d['ms_per_step'],d['stage_ms'])"
if [ -n "$KREGEX" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" --launch-skip ${SKIP:-6} -c ${COUNT:-2} -o gpurun_out/${OUT:-prof} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${OUT:-prof}.log 2>&1; echo ncu=$?
fi
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo launches=$?
fi
