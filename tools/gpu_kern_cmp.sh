# per-kernel ncu metrics (1 tick after warm-up) for alternative library builds: LIBS, KREGEX, WL, METRICS
M=${METRICS:-gpu__time_duration.sum}
for L in ${LIBS}; do echo "LIB=$L"; TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/$L timeout 300 ncu --metrics $M --clock-control none -k "regex:${KREGEX}" --launch-skip ${SKIP:-12} -c ${COUNT:-6} --csv python bench.py --workload ${WL:-C5} --no-cpu-baseline --no-e2e --steps 2 --warmup 3 2>/dev/null | grep -E "^\"[0-9]+\",.*(${KREGEX})" | awk -F'","' '{print $5, $(NF-2), $NF}'; done
