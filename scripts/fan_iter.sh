#!/bin/bash
# One fan-kernel iteration on the GPU box: EBE parity tests, variant timing, ncu capture (tag = $1).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-fan}
timeout 600 python -m pytest tests/test_ebe_gpu.py tests/test_unstructured_gpu.py -m gpu -x -q > gpurun_out/${tag}_tests.txt 2>&1
timeout 300 python scripts/ebe_time.py pair,fan > gpurun_out/${tag}_time.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_ebe_fan -s 3 -c 1 -o gpurun_out/${tag} python scripts/ebe_once.py 32 2 16 > /dev/null 2>&1
tail -2 gpurun_out/${tag}_tests.txt; grep -v "^\[" gpurun_out/${tag}_time.txt | head -20
