set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
nproc; free -g | head -2
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum -k regex:lambda_tuned -c 4 --csv --log-file gpurun_out/ncu_tuned_write.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu > /dev/null 2>&1; echo ncu_rc=$?
tail -5 gpurun_out/pytest_gpu.log
