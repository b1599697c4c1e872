# Builds K5 variant libraries build/k5v/lib_G<g>_U<u>.so (column group size x
# record-loop unroll) for A/B timing with SP_LIB=... python tools/k5_time.py.
#   bash tools/k5_variants.sh "8 1" "8 2" "4 3"
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2311_03906_b200/csrc >/dev/null
O=build/obj; V=build/k5v; mkdir -p $V
for gu in "$@"; do
  set -- $gu
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
    -DK5_G=$1 -DK5_UNR=$2 -c paper_2311_03906_b200/csrc/k5_columns.cu -o $V/k5_G$1_U$2.o &
done
wait
for f in $V/k5_G*.o; do
  t=${f#$V/k5_}; t=${t%.o}
  objs=$(ls $O/*.o | grep -v k5_columns.o)
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $V/lib_$t.so $objs $f -Xcompiler -fPIC -cudart static
done
ls -la $V/*.so
