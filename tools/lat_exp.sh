o=gpurun_out/${1:-lat}; mkdir -p $o
for m in 0 16 48 2; do for pp in 0 1; do
SP_AUTOTUNE=0 SP_GEN_WARPS=12 SP_PAD_PRED=$pp SP_DEBUG_MODE=$m python tools/time_kernel.py --config cfg3 --shots 10000000 --tiled --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 mode=$m pp=$pp', round(d['ms_median'],4))" >> $o/t.txt 2>&1
SP_AUTOTUNE=0 SP_GEN_WARPS=10 SP_PAD_PRED=$pp SP_DEBUG_MODE=$m python tools/time_kernel.py --config cfg2 --shots 10002432 --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 mode=$m pp=$pp', round(d['ms_median'],4))" >> $o/t.txt 2>&1
done; done
cat $o/t.txt
