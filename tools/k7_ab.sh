# A/B of env switches for K1 and K7 at cfg3 (tiled, detector counts) and cfg2.
o=gpurun_out/${1:-k7ab}; mkdir -p $o
run() { cfg="$1"; shift; env "$@" timeout 160 python tools/k7_check.py $cfg --reps 5 2>>$o/err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config'], 'tiled' if d['tiled'] else 'mm', ' '.join(f'{k}={v}' for k,v in d['env'].items() if k!='SP_QUEUED'), 'identical', d['identical'], 'k1', round(d['k1_ms'],4), 'k7', round(d['k7_ms'],4))" >> $o/t.txt; }
for tex in 1 0; do
run "--config cfg3 --shots 10000000 --tiled --dets" SP_LIST_TEX=$tex SP_Q_WALK=8 SP_Q_APPLY=8
run "--config cfg3 --shots 10000000 --tiled --dets" SP_LIST_TEX=$tex SP_Q_WALK=12 SP_Q_APPLY=12 SP_Q_DEPTH=4
run "--config cfg2 --shots 10002432" SP_LIST_TEX=$tex SP_Q_WALK=8 SP_Q_APPLY=8
run "--config cfg3 --shots 10000000 --tiled" SP_LIST_TEX=$tex SP_Q_WALK=8 SP_Q_APPLY=8
done
cat $o/t.txt
