# parity subset + timings of cfg3 (tiled) / cfg2 (mm) with no counts, measurement counts, detector counts
o=gpurun_out/${1:-aa}; mkdir -p $o
[ -n "$TESTS" ] && { timeout 900 python -m pytest tests -m gpu -x -q -k "$TESTS" > $o/tests.log 2>&1; tail -2 $o/tests.log; }
for cfg in "cfg3 --shots 10000000 --tiled" "cfg2 --shots 10002432"; do
for x in "" "--counts" "--dets"; do
env $ENVS python tools/time_kernel.py --config $cfg $x --reps 9 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $x', round(d['ms_median'],4), d['plan']['gen_warps'])" >> $o/t.txt 2>&1
done; done
cat $o/t.txt
