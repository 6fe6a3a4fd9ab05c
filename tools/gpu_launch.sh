# launch list of the bench workload (last frames) + a bench line
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_probe.py 10 > gpurun_out/ncu_probe.log 2>&1
tail -1 gpurun_out/ncu_probe.log
timeout 600 python bench.py --steps 20 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
