# element-order slab count: kernel time, DRAM traffic (ncu) and e2e of the host-buffer apply
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for s in 1 8 16 32; do
  echo "SLABS=$s"
  TSGPU_EBE_SLABS=$s timeout 300 python scripts/ebe_time.py pair 82,123,41 2>&1 | grep -E "fp32_r(1|16)_pair|o1_fp32"
  TSGPU_EBE_SLABS=$s timeout 300 python bench.py --steps 30 --no-sweep --no-cpu-baseline --no-greens --no-solve 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('value', d['value'], 'e2e', d['e2e']['value'], 'kernel_ms', d['roofline']['kernel_ms'])"
  TSGPU_EBE_SLABS=$s timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_ebe_pair -s 3 -c 1 python scripts/ebe_once.py 32 2 16 2>&1 | grep -E "dram__bytes"
done
