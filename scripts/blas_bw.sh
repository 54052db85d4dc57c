# DRAM bandwidth of the PCG streaming passes in a configs[1]-size solve (ncu, per launch); the longest
# launches of each kernel are the level-0 ones
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file gpurun_out/blas_bw.csv -k regex:"k_update|k_direction|k_gamma|k_bcsr_rows" -c 1500 \
  python scripts/solve_time.py 82,123,41 16 > /dev/null 2>&1
echo rc=$?
