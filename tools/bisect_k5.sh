for e in "-" "SP_SEG_STAGE=0" "SP_BULK=0" "SP_SEG_STAGE=0 SP_BULK=0" "SP_AUTOTUNE=0"; do
  [ "$e" = "-" ] && ev="" || ev="$e"
  echo "== $e"; env $ev timeout 300 python -m pytest tests/test_gpu_k5.py -x -q 2>&1 | tail -1
done
