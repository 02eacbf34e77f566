#!/bin/bash
# summarise gpurun_out/prof_tc.ncu-rep here (no GPU needed)
R=${1:-gpurun_out/prof_tc.ncu-rep}
ncu -i $R --page raw --csv > /tmp/raw.csv 2>/dev/null
ncu -i $R --page source --csv --print-source cuda,sass > /tmp/src.csv 2>/dev/null
python - <<'PY'
import csv
r=list(csv.reader(open('/tmp/raw.csv'))); h=r[0]; d=dict(zip(h,r[-1]))
for k in ['gpu__time_duration.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active',
 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed','l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum.pct_of_peak_sustained_elapsed',
 'l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
 'smsp__inst_executed.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct','launch__registers_per_thread']:
    print(f"{k:80s} {d.get(k)}")
out=[]
for k in h:
    if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
        try: out.append((float(d[k].replace(',','')),k[33:]))
        except: pass
s=sum(v for v,k in out)
print('stalls:', ' '.join(f"{k}:{100*v/s:.0f}%" for v,k in sorted(out,reverse=True)[:10]))
PY
python tools/ncu_source_top.py /tmp/src.csv 20
