#!/bin/bash
# A/B of the MUSIC spectrum paths on C4 (development aid): SSLG_SPECTRUM_TC=0
# (FP64 DMMA) vs 1 (tcgen05 kind::tf32 3-pass), bench spectrum time per launch.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for v in 0 1; do
  SSLG_SPECTRUM_TC=$v timeout 300 python bench.py --config c4 --steps 5 --no-cpu-baseline > gpurun_out/c4_tc$v.json 2>gpurun_out/c4_tc$v.err
  python - <<PY
import json
d = json.loads(open("gpurun_out/c4_tc$v.json").read().strip().splitlines()[-1])
k = d["kernels"]["spectrum"]
print("TC=$v blocks/s", round(d["value"], 1), "spectrum us/block", round(1e3 * k["ms_per_launch"] / 32, 1),
      "hits", d["target_hit_rate"])
PY
done
