#!/bin/bash
# Launch-size sweep of the pair sweep (TSGPU_EBE_PAIR_STRIDES) at configs[3] (one device) and configs[1].
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for s in ${CFG3_STRIDES:-0 256 512 1024}; do
  TSGPU_EBE_PAIR_STRIDES=$s timeout 300 python scripts/maxsize_bench.py --steps 8 > gpurun_out/st_cfg3_$s.json 2> gpurun_out/st_cfg3_$s.err
  echo "cfg3 strides=$s $(python -c "import json;d=json.load(open('gpurun_out/st_cfg3_$s.json'));print(d['fp32_r8']['kernel_ms'],d['fp32_r4']['kernel_ms'])" 2>&1 | tail -1)"
done
for s in ${CFG2_STRIDES:-0 256}; do
  TSGPU_EBE_PAIR_STRIDES=$s timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-solve --no-greens --steps 50 > gpurun_out/st_cfg2_$s.json 2> gpurun_out/st_cfg2_$s.err
  echo "cfg2 strides=$s $(python -c "import json;d=json.loads(open('gpurun_out/st_cfg2_$s.json').read().splitlines()[-1]);print(d['roofline']['kernel_ms'],d['ms_per_step'],d['e2e']['ms_per_step'])" 2>&1 | tail -1)"
done
