#!/bin/bash
# One tiled-fan iteration on the GPU box: tiled-fan parity tests, variant timing, ncu capture (tag = $1).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-fantile}
timeout 600 python -m pytest tests/test_ebe_gpu.py tests/test_unstructured_gpu.py -m gpu -x -q -k "fantile" > gpurun_out/${tag}_tests.txt 2>&1
timeout 300 python scripts/ebe_time.py pair,fan,fantile > gpurun_out/${tag}_time.txt 2>&1
TSGPU_EBE_KERNEL=fantile timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_ebe_fantile -s 3 -c 1 -o gpurun_out/${tag} python scripts/ebe_once.py 32 2 16 > /dev/null 2>&1
tail -3 gpurun_out/${tag}_tests.txt; grep -v "^\[" gpurun_out/${tag}_time.txt | head -20
