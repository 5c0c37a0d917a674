# Experiment builds that differ in ONE kernel file (seconds, not minutes):
#   bash tools/build_file_variant.sh name qg_short.cu [-Dflags]  -> _lib/var_name/libqgemm_b200.so (QG_LIB_PATH)
set -e
name=$1; file=$2; shift; shift
here=$(cd "$(dirname "$0")/.." && pwd)
out=$here/paper_0803_1975_b200/_lib/var_$name
mkdir -p "$out" /tmp/qg_fv_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -Xptxas -v "$@" \
  -c -o /tmp/qg_fv_$name/$file.o $here/paper_0803_1975_b200/csrc/$file 2> /tmp/qg_fv_$name/ptxas.log
objs=$(ls $here/paper_0803_1975_b200/build/*.o | grep -v "/$file.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libqgemm_b200.so $objs /tmp/qg_fv_$name/$file.o -lcudart -ldl
echo built $out/libqgemm_b200.so
