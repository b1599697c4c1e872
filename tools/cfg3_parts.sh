# cfg3 K1 time with parts switched off (SP_DEBUG_MODE bits: 1 XORs, 2 walks, 4 coins, 8 drain)
o=gpurun_out/${1:-parts}; mkdir -p $o
for m in ${4:-0 1 4 8 2 6 9 10 12 14}; do
SP_DEBUG_MODE=$m timeout 120 python tools/time_kernel.py --config ${2:-cfg3} --shots ${3:-10000000} --tiled --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode=$m', round(d['ms_median'],4), d['plan']['gen_warps'])" >> $o/parts.txt 2>&1
done
cat $o/parts.txt
