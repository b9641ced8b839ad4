# ncu --set full of selected kernels on a short bench run: KREGEX, SKIP, COUNT, OUT
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_join}" \
  --launch-skip ${SKIP:-3} -c ${COUNT:-1} -o gpurun_out/${OUT:-prof} \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/${OUT:-prof}.log 2>&1
echo ncu=$?
tail -3 gpurun_out/${OUT:-prof}.log
