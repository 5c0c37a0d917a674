# Experiment builds that differ only in qg_anchor.cu (seconds, not minutes):
#   bash tools/build_anchor_variant.sh name [-Dflags]  -> _lib/var_name/libqgemm_b200.so (QG_LIB_PATH)
set -e
name=$1; shift
here=$(cd "$(dirname "$0")/.." && pwd)
out=$here/paper_0803_1975_b200/_lib/var_$name
mkdir -p "$out" /tmp/qg_av_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -Xptxas -v "$@" \
  -c -o /tmp/qg_av_$name/qg_anchor.cu.o $here/paper_0803_1975_b200/csrc/qg_anchor.cu 2> /tmp/qg_av_$name/ptxas.log
objs=$(ls $here/paper_0803_1975_b200/build/*.o | grep -v qg_anchor)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libqgemm_b200.so $objs /tmp/qg_av_$name/qg_anchor.cu.o -lcudart -ldl
grep -A1 "Function properties" /tmp/qg_av_$name/ptxas.log | grep "spill" | tr '\n' ';'; echo; echo built $out/libqgemm_b200.so
