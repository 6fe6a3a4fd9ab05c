#!/bin/bash
# GPU box, end of round: the full -m gpu suite with the parity report, the
# driver-contract bench lines of every config, the reference arm, a 2-rank run on
# one GPU, the ncu launch list of the default bench command and one ncu --set
# full capture of a frame (all kernels) for the per-family DRAM traffic.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/smi_final.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  DFX_PARITY_REPORT=gpurun_out/parity_final.json timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests_final.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/gpu_tests_final.log; tail -4 gpurun_out/gpu_tests_final.log
  (cd .refsmoke 2>/dev/null && PYTHONPATH=$GRAFT_REPO_ROOT timeout 300 python -m pytest test_smoke.py -q -rA -p no:cacheprovider > ../gpurun_out/smoke_ref_final.log 2>&1; echo "rc=$?" >> ../gpurun_out/smoke_ref_final.log)
fi
timeout 900 python bench.py > gpurun_out/bench_c2_final.log 2>&1; echo "c2 rc=$?"
for c in c3 c4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_final.log 2>&1; echo "$c rc=$?"; done
timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 10 > gpurun_out/bench_c5_final.log 2>&1; echo "c5 rc=$?"
timeout 900 python bench.py --gpus 2 --no-cpu-baseline --no-sweep > gpurun_out/bench_c2_2ranks_1gpu.log 2>&1; echo "2ranks rc=$?"
for s in 1 2 4 8; do timeout 600 python bench.py --streams $s --no-cpu-baseline --no-sweep > gpurun_out/bench_c2_streams$s.log 2>&1; echo "streams $s rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -s 186 -c 31 -o gpurun_out/frame_full \
  python tools/ncu_probe.py 8 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/frame_full.ncu-rep --page raw --csv > gpurun_out/frame_full_raw.csv 2>/dev/null; ls -la gpurun_out/frame_full.ncu-rep; [ $(stat -c %s gpurun_out/frame_full.ncu-rep) -gt 40000000 ] && rm -f gpurun_out/frame_full.ncu-rep
if [ -z "$SKIP_REF" ]; then
  timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_final.log 2>&1; echo "ref rc=$?"
fi
ls -la gpurun_out | tail -30
