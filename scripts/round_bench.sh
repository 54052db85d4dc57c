#!/bin/bash
# Full 1-GPU bench + reference arm + launch list of the bench's timed kernels.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?" >> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-solve > /dev/null 2>&1
tail -2 gpurun_out/bench_full.err; cat gpurun_out/bench_full.json | cut -c1-1500; cat gpurun_out/bench_ref.json | cut -c1-400
