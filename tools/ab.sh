# A/B timing of the fused sampler: bash tools/ab.sh TAG "ENV1" "ENV2" ...   (ENV "-" = defaults)
o=gpurun_out/$1; shift; mkdir -p $o
[ -n "$TESTS" ] && { timeout 900 python -m pytest tests -m gpu -x -q -k "$TESTS" > $o/tests.log 2>&1; tail -2 $o/tests.log; }
for e in "$@"; do
for cfg in "cfg3 --shots 10000000 --tiled" "cfg2 --shots 10002432" "cfg4 --shots 1000000 --tiled"; do
  [ "$e" = "-" ] && ev="" || ev="$e"
  env $ev python tools/time_kernel.py --config $cfg --reps ${REPS:-7} | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e] $cfg', round(d['ms_median'],4), 'gw', d['plan']['gen_warps'], 'pp', d['plan']['pad_pred'])" >> $o/t.txt 2>&1
done; done
cat $o/t.txt
