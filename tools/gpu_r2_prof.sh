# decode list-shape distribution at C5 + ncu --set full of the join and the decode
mkdir -p gpurun_out
timeout 600 python tools/decode_profile.py C5 > gpurun_out/decode_profile.log 2>&1
KREGEX="k_decode_query|k_join|k_query_fill" SKIP=9 COUNT=3 OUT=prof_r2b bash tools/gpu_prof.sh
