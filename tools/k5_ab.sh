# A/B the K5 variant libraries built by tools/k5_variants.sh on cfg5 shapes.
o=gpurun_out/${1:-k5ab}; mkdir -p $o
for lib in build/k5v/lib_*.so; do
  for dp in "0.5 1e-3" "0.5 1e-2" "0.5 1e-4" "0.01 1e-3"; do
    echo "$(basename $lib) $(SP_LIB=$PWD/$lib python tools/k5_time.py $dp 2>&1 | tail -1)"
  done
done > $o/t.txt
