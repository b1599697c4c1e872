# A/B of one env switch on K1 (and K7) at cfg3 tiled with detector counts: tools/ab_env.sh NAME VAR v1 v2 ...
o=gpurun_out/${1:-abe}; var=$2; shift 2; mkdir -p $o
for v in "$@"; do
env $var=$v timeout 160 python tools/k7_check.py --config cfg3 --shots 10000000 --tiled --dets --reps 5 2>>$o/err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$var=$v', 'identical', d['identical'], 'k1', round(d['k1_ms'],4), 'k7', round(d['k7_ms'],4), 'gw', d['res']['k1']['plan']['gen_warps'])" >> $o/t.txt
done
cat $o/t.txt
