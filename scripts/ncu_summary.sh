#!/bin/bash
# usage: scripts/ncu_summary.sh report.ncu-rep  -> key SOL / memory / stall metrics
R=$1
ncu -i $R --page details --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keep=('GPU Speed','Memory Workload','Scheduler','Warp State','Occupancy','Launch','Compute Workload')
for row in r[1:]:
    d=dict(zip(h,row))
    if d.get('Section Name','').startswith(keep) and d.get('Metric Name'):
        print(d['Section Name'][:18], '|', d['Metric Name'][:48], '|', d['Metric Value'], d.get('Metric Unit',''))
"
ncu -i $R --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; u=r[1]; v=r[2]
out=[]
for a,b,c in zip(h,u,v):
    if a.startswith('smsp__pcsamp_warps_issue_stalled_') and not a.endswith('not_issued'):
        out.append((float(c or 0), a.replace('smsp__pcsamp_warps_issue_stalled_','stall_'), b))
    elif a in ('dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sectors_srcunit_tex_op_read.sum','lts__t_sectors_srcunit_tex_op_write.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum','smsp__inst_executed.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','launch__registers_per_thread'):
        out.append((1e30, a, c+' '+b))
for x in sorted(out, key=lambda z:-z[0])[:40]:
    print(x[1], x[2] if x[0]==1e30 else int(x[0]))
"
