# Experiment builds of the library with extra nvcc defines, e.g.
#   bash tools/build_variant.sh sg8 -DQG_SPLIT_GROUPS=8
# -> paper_0803_1975_b200/_lib/var_sg8/libqgemm_b200.so (select with QG_LIB_PATH)
set -e
name=$1; shift
here=$(cd "$(dirname "$0")/.." && pwd)
out=$here/paper_0803_1975_b200/_lib/var_$name
bld=/tmp/qg_var_$name
mkdir -p "$out" "$bld"
flags="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr $*"
objs=""
for f in qg_abi.cu qg_dot.cu qg_small.cu qg_anchor.cu qg_pack.cu qg_word64.cu; do
  nvcc $flags -c -o $bld/$f.o $here/paper_0803_1975_b200/csrc/$f &
  objs="$objs $bld/$f.o"
done
for f in qg_plan.cpp qg_io.cpp qg_multi.cpp qg_stage.cpp; do
  nvcc $flags -x cu -c -o $bld/$f.o $here/paper_0803_1975_b200/csrc/$f &
  objs="$objs $bld/$f.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libqgemm_b200.so $objs -lcudart -ldl
echo built $out/libqgemm_b200.so
