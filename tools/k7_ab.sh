# A/B of env switches for K1 and K7 at cfg3 (tiled, detector counts) and cfg2.
o=gpurun_out/${1:-k7ab}; mkdir -p $o
run() { cfg="$1"; shift; env "$@" timeout 160 python tools/k7_check.py $cfg --reps 5 2>>$o/err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config'], 'tiled' if d['tiled'] else 'mm', 'dets' if d['dets'] else '', ' '.join(f'{k}={v}' for k,v in d['env'].items() if k!='SP_QUEUED'), 'identical', d['identical'], 'k1', round(d['k1_ms'],4), 'k7', round(d['k7_ms'],4))" >> $o/t.txt; }
for shape in "8 8 8" "12 12 4" "10 10 8" "12 12 8" "14 14 4" "8 16 8" "10 10 4"; do
set -- $shape
run "--config cfg3 --shots 10000000 --tiled --dets" SP_Q_WALK=$1 SP_Q_APPLY=$2 SP_Q_DEPTH=$3
done
run "--config cfg3 --shots 10000000 --tiled" SP_Q_WALK=12 SP_Q_APPLY=12 SP_Q_DEPTH=4
run "--config cfg2 --shots 10002432" SP_Q_WALK=12 SP_Q_APPLY=12 SP_Q_DEPTH=4
run "--config cfg2 --shots 10002432" SP_Q_WALK=8 SP_Q_APPLY=8 SP_Q_DEPTH=8
cat $o/t.txt
