o=gpurun_out/${1:-abd}; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_detcounts.py -x -q > $o/tests.log 2>&1; tail -2 $o/tests.log
for cfg in "cfg3 --shots 10000000 --tiled"; do
for x in "" "--counts" "--dets"; do for m in 0 2; do
SP_DEBUG_MODE=$m python tools/time_kernel.py --config $cfg $x --reps 9 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $x mode=$m', round(d['ms_median'],4), d['plan']['gen_warps'])" >> $o/t.txt 2>&1
done; done; done
cat $o/t.txt
