#!/bin/bash
# One GPU session: parity tests, bench (C3 + C4), launch list, full ncu
# captures of the top kernels.  Outputs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
STEPS=${STEPS:-10}
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -2 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py --steps $STEPS > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --config c4 --steps 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "bench c4 rc=$?"
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --batch 8 --no-cpu-baseline --no-flush > gpurun_out/ncu_launch.log 2>&1
  echo "ncu launches rc=$?"
  # the split solver: per push jacobi_kernel<60,1>, sweep_kernel, jacobi_kernel<60,3>
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^jacobi_kernel" -s 2 -c 1 \
    -o gpurun_out/prof_jacobi_prologue -f python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-flush \
    > gpurun_out/ncu_jacobi_prologue.log 2>&1
  echo "ncu jacobi prologue rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^jacobi_kernel" -s 3 -c 1 \
    -o gpurun_out/prof_jacobi_epilogue -f python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-flush \
    > gpurun_out/ncu_jacobi_epilogue.log 2>&1
  echo "ncu jacobi epilogue rc=$?"
  for K in ${NCU_KERNELS:-sweep_kernel spectrum_mma_kernel correlation_kernel stft_kernel canonical_kernel}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 1 -c 1 \
      -o gpurun_out/prof_$K -f python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-flush \
      > gpurun_out/ncu_$K.log 2>&1
    echo "ncu $K rc=$?"
  done
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spectrum_mma -s 1 -c 1 \
    -o gpurun_out/prof_spectrum_mma_c4 -f python bench.py --config c4 --steps 1 --warmup 1 --batch 8 \
    --no-cpu-baseline --no-flush > gpurun_out/ncu_spectrum_mma_c4.log 2>&1
  echo "ncu spectrum_mma c4 rc=$?"
fi
