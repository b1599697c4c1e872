o=gpurun_out/${1:-abn2}; mkdir -p $o
for e in "SP_NBUF=2" "SP_NBUF=3" "SP_NBUF=3 SP_LIST_TEX=0" "SP_NBUF=3 SP_ROWSTAGED=0" "SP_NBUF=3 SP_Q_DEPTH=2"; do
env $e timeout 160 python tools/k7_check.py --config cfg3 --shots 10000000 --tiled --dets --reps 5 --no-check 2>>$o/err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$e', 'k1', round(d['k1_ms'],4), d['res']['k1']['plan']['smem_bytes'], 'k7', round(d['k7_ms'],4), d['res']['k7']['plan']['fused_ok'])" >> $o/t.txt
done
cat $o/t.txt
