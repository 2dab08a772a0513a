#!/bin/bash
# The round's measurement record on one B200: tools/gpu_round.sh (tests,
# C3/C4 bench, ncu) plus C1, C2, C5, bin sharding and the reference arm.
# Outputs in gpurun_out/; copy into profiles/<round>/ (see profiles/r01/README.md).
cd "${GRAFT_REPO_ROOT}"
SKIP_TESTS=0 bash tools/gpu_round.sh
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/b_c1.json 2>gpurun_out/b_c1.err; echo c1 $?
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b_c2.json 2>gpurun_out/b_c2.err; echo c2 $?
timeout 600 python bench.py --arrays 64 --batch 8 --steps 3 --no-cpu-baseline > gpurun_out/b_c5.json 2>gpurun_out/b_c5.err; echo c5 $?
timeout 300 python bench.py --shard bins --steps 5 --no-cpu-baseline > gpurun_out/b_bs.json 2>gpurun_out/b_bs.err; echo bs $?
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b_ref.json 2>gpurun_out/b_ref.err; echo ref $?
