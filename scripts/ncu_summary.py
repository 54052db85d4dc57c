"""Key metrics of an ncu report (details + stall reasons + dram bytes)."""
import csv, subprocess, sys
def page(rep, p):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))
for rep in sys.argv[1:]:
    print("===", rep)
    rows = page(rep, "details"); hdr = rows[0]
    keep = ['Duration','DRAM Throughput','L2 Cache Throughput','L1/TEX Cache Throughput','Compute (SM) Throughput',
            'Achieved Occupancy','Registers Per Thread','Executed Ipc Active','Issue Slots Busy','L2 Hit Rate',
            'Warp Cycles Per Issued Instruction','Executed Instructions','SM Frequency','Dynamic Shared Memory Per Block']
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get('Metric Name') in keep:
            print(f"  {d['Metric Name']:36s} {d['Metric Value']:>14s} {d['Metric Unit']}")
    rows = page(rep, "raw"); hdr, vals = rows[0], rows[2]
    d = dict(zip(hdr, vals))
    for k in ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
              'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active']:
        print(f"  {k:60s} {d.get(k)}")
    st = [(h.replace('smsp__pcsamp_warps_issue_stalled_', ''), float(v.replace(',', ''))) for h, v in d.items()
          if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued')]
    tot = sum(v for _, v in st) or 1
    print("  stalls: " + ", ".join(f"{h} {100*v/tot:.0f}%" for h, v in sorted(st, key=lambda x: -x[1])[:7]))
