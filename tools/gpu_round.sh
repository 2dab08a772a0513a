#!/bin/bash
# One GPU session of measurements for the round record: parity tests, the
# bench lines of every BASELINE config, the ncu launch list of the headline
# command, and one `ncu --set full` capture per hot kernel and config
# (files prof_<config>__<kernel>.ncu-rep -> tools/ncu_summary.py -> the
# per-config DRAM traffic bench.py reports).  Outputs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
STEPS=${STEPS:-10}
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -2 gpurun_out/pytest_gpu.log
  ./tests/cpp/test_dropin.bin > gpurun_out/cpp_dropin.log 2>&1; echo "cpp drop-in rc=$?"
fi
timeout 900 python bench.py --steps $STEPS > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench c3 rc=$?"
for c in c1 c2 c4; do
  timeout 900 python bench.py --config $c --steps $STEPS --cpu-sample-blocks 8 > gpurun_out/bench_$c.json \
    2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py --arrays 64 --batch 8 --steps 3 --no-cpu-baseline > gpurun_out/bench_c5.json \
  2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
timeout 300 python bench.py --shard bins --steps 5 --no-cpu-baseline > gpurun_out/bench_binshard.json \
  2> gpurun_out/bench_binshard.err; echo "bench bin-shard rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json \
  2> gpurun_out/bench_reference.err; echo "reference arm rc=$?"
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --batch 8 --no-cpu-baseline --no-flush > gpurun_out/ncu_launch.log 2>&1
  echo "ncu launches rc=$?"
  cap() {  # cap <config> <name> <kernel regex> <skip> [extra bench args]
    local cfg=$1 name=$2 rx=$3 skip=$4; shift 4
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s "$skip" -c 1 \
      -o "gpurun_out/prof_${cfg}__${name}" -f python bench.py --config "$cfg" --steps 1 --warmup 1 --batch "$@" \
      --no-cpu-baseline --no-flush > "gpurun_out/ncu_${cfg}__${name}.log" 2>&1
    echo "ncu $cfg $name rc=$?"
  }
  # the split solver at m = 60: per push jacobi_kernel<60,1>, sweep_bip_kernel, jacobi_kernel<60,3>
  cap c3 jacobi_prologue "^jacobi_kernel" 2 8
  cap c3 jacobi_epilogue "^jacobi_kernel" 3 8
  for K in sweep_bip_kernel spectrum_mma_kernel correlation_kernel stft_kernel integrate_peaks_kernel; do
    cap c3 $K "^$K" 1 8
  done
  cap c4 spectrum_tc_kernel "^spectrum_tc_kernel" 1 8
  cap c1 small_jacobi_kernel "^small_jacobi_kernel" 1 4
  cap c2 small_jacobi_kernel "^small_jacobi_kernel" 1 4
  # summaries on the box (the reports exceed gpurun's 64 MiB copy-back):
  # text per capture, launch shares, per-config DRAM traffic
  python tools/ncu_summary.py r02 gpurun_out/summary > /dev/null 2>&1; echo "ncu summary rc=$?"
  mkdir -p gpurun_out/reps
  for f in gpurun_out/prof_c3__sweep_bip_kernel gpurun_out/prof_c3__jacobi_epilogue gpurun_out/prof_c4__spectrum_tc_kernel; do
    [ -f $f.ncu-rep ] && mv $f.ncu-rep gpurun_out/reps/
  done
  rm -f gpurun_out/prof_*.ncu-rep
fi
