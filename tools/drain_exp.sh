o=gpurun_out/${1:-de}; mkdir -p $o
for e in "SP_DEBUG_MODE=2" "SP_DEBUG_MODE=2 SP_BULK=0" "SP_DEBUG_MODE=2 SP_WAIT_NS=32" "SP_DEBUG_MODE=6" "SP_DEBUG_MODE=6 SP_BULK=0" "SP_DEBUG_MODE=14" "SP_DEBUG_MODE=14 SP_BULK=0" "SP_DEBUG_MODE=10" "SP_WAIT_NS=32" "SP_WAIT_NS=64"; do
env $e SP_AUTOTUNE=0 SP_GEN_WARPS=10 python tools/time_kernel.py --config cfg3 --shots 10000000 --tiled --reps 7 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e]', round(d['ms_median'],4))" >> $o/t.txt 2>&1
done
cat $o/t.txt
