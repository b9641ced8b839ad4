# bench each library variant (LIBS = file names under paper_1411_3212_b200/_lib/), short runs
for L in ${LIBS}; do
  echo "== $L" >> gpurun_out/variants.log
  TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/$L timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} 2>&1 | python -c "
import json,sys
for x in sys.stdin:
  if x.startswith('{'):
    d=json.loads(x); print(round(d['value']/1e9,4), 'Gq/s p50', round(d['p50_tick_ms'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, 'join_frac', round(d['roofline']['frac'],3), 'k1_ms', round(d['roofline_index']['ms'],3))
  elif 'rror' in x: print(x.strip()[:300])
" >> gpurun_out/variants.log
done
