o=gpurun_out/mb; mkdir -p $o
./build/mb_atoms > $o/mb_atoms.jsonl 2>&1
for pp in 0 1; do for gw in 10 11 12 13; do
SP_AUTOTUNE=0 SP_PAD_PRED=$pp SP_GEN_WARPS=$gw python tools/time_kernel.py --config cfg3 --shots 10000000 --tiled --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pp=$pp gw=$gw', d['ms_median'])" >> $o/cfg3_sweep.txt 2>&1
done; done
cat $o/mb_atoms.jsonl $o/cfg3_sweep.txt
