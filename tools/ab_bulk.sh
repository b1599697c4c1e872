o=gpurun_out/${1:-ab}; mkdir -p $o
[ -n "$NOTEST" ] || timeout 600 python -m pytest tests -m gpu -x -q -k "parity or large or detectors or k5 or stats" > $o/tests.log 2>&1; tail -3 $o/tests.log
for cfg in "cfg3 --shots 10000000 --tiled" "cfg2 --shots 10002432" "cfg2 --shots 10002432 --counts" "cfg3 --shots 10000000 --tiled --counts" "cfg4 --shots 1000000 --tiled"; do
for bk in 0 1; do
SP_BULK=$bk python tools/time_kernel.py --config $cfg --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg bulk=$bk', round(d['ms_median'],4), d['plan']['gen_warps'])" >> $o/t.txt 2>&1
done; done
cat $o/t.txt
