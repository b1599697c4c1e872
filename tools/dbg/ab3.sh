# A/B of two builds on cfg2 / cfg3 (tools/sweep_env.sh) and cfg4 (tiled)
a=$1; b=$2
bash tools/sweep_env.sh "SP_LIB=$a" "SP_LIB=$b" "SP_LIB=$a" "SP_LIB=$b"
for l in $a $b; do SP_LIB=$l python tools/time_kernel.py --config cfg4 --counts --tiled --reps 10 | python -c "import json,sys; d=json.load(sys.stdin); print('$l cfg4', round(d['ms_median'],4))"; done
