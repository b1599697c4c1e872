#!/bin/bash
# Ad-hoc variant sweep: each argument is "ENV=.. ENV=.. -- time_kernel args".
out=gpurun_out/sweep2.jsonl
: > $out
T="python tools/time_kernel.py"
for spec in "$@"; do
  envs="${spec%%--*}"; args="${spec#*--}"
  timeout 120 env $envs $T $args >> $out 2>>gpurun_out/sweep2.err
done
python - <<'PY'
import json
for l in open("gpurun_out/sweep2.jsonl"):
    d = json.loads(l)
    p = d["plan"]
    print(f'{d["config"]:5s} tiled={int(d["tiled"])} counts={int(d.get("counts", 0))} {d["env"]} ms={d["ms_median"]:.4f} GBps={d["GBps"]:.0f} '
          f'T={p["shot_tile"]} gw={p["gen_warps"]} seg={p["n_segments"]} lp={p["lp"]} pp={p["pad_pred"]}'
          + (f' timers={d["timers"]}' if d.get("timers") else ''))
PY
