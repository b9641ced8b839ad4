# Build an experimental library variant: bash tools/build_variant.sh NAME [-DMACRO=V ...]
# -> paper_1411_3212_b200/_lib/exp_NAME.so (select at run time with TJ_LIB_PATH)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC -shared \
  -I include "$@" -o paper_1411_3212_b200/_lib/exp_$name.so paper_1411_3212_b200/csrc/tj_abi.cu
