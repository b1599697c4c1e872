# A/B of an alternative library build: bash tools/ab_lib.sh TAG LIBPATH
o=gpurun_out/$1; mkdir -p $o
for lib in "" "$2"; do
for cfg in "cfg3 --shots 10000000 --tiled" "cfg3 --shots 10000000 --tiled --dets" "cfg2 --shots 10002432" "cfg4 --shots 1000000 --tiled"; do
  SP_LIB=$lib python tools/time_kernel.py --config $cfg --reps 9 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[${lib:-default}] $cfg', round(d['ms_median'],4), 'gw', d['plan']['gen_warps'], 'pp', d['plan']['pad_pred'])" >> $o/t.txt 2>&1
done; done
cat $o/t.txt
