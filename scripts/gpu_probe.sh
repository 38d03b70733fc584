set -x
./scripts/probe_partial > gpurun_out/probe.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum --csv --log-file gpurun_out/probe_ncu.csv ./scripts/probe_partial > /dev/null 2>&1
echo done
