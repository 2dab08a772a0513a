#!/bin/bash
# One GPU session: parity tests, bench, launch list, full ncu capture of the
# top kernel(s).  Outputs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
STEPS=${STEPS:-10}
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py --steps $STEPS > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --batch 8 --no-cpu-baseline --no-flush > gpurun_out/ncu_launch.log 2>&1
  echo "ncu launches rc=$?"
  for K in ${NCU_KERNELS:-jacobi_kernel canonical_kernel spectrum_kernel}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o gpurun_out/prof_$K -f python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-flush \
      > gpurun_out/ncu_$K.log 2>&1
    echo "ncu $K rc=$?"
  done
fi
