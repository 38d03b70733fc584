# usage: bash scripts/gpu_round.sh TAG [tests] [bench] [stencil] [ncu] [ncufull]
TAG=$1; shift
mkdir -p gpurun_out/$TAG
for step in "$@"; do
case $step in
tests)
  timeout 300 python __graft_entry__.py smoke > gpurun_out/$TAG/smoke.log 2>&1; echo smoke_rc=$?
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo pytest_rc=$?
  tail -3 gpurun_out/$TAG/pytest_gpu.log ;;
bench)
  timeout 900 python bench.py > gpurun_out/$TAG/bench_write16.json 2> gpurun_out/$TAG/bench_write16.err; echo bench_rc=$?
  timeout 600 python bench.py --impl reference > gpurun_out/$TAG/bench_ref.json 2> gpurun_out/$TAG/bench_ref.err; echo ref_rc=$? ;;
stencil)
  timeout 900 python bench.py --workload stencil17 --steps 100 > gpurun_out/$TAG/bench_stencil17.json 2> gpurun_out/$TAG/bench_stencil17.err; echo stencil_rc=$? ;;
ncu)
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/$TAG/launches_write16.csv python bench.py --steps 20 --warmup 3 --no-sweep --no-e2e --no-cpu > /dev/null 2>&1; echo ncu_rc=$?
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/$TAG/launches_stencil17.csv python bench.py --workload stencil17 --steps 10 --warmup 3 --no-sweep --no-e2e --no-cpu > /dev/null 2>&1; echo ncu2_rc=$? ;;
ncufull)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gasket_write -s 3 -c 1 -o gpurun_out/$TAG/prof_write16 python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu > /dev/null 2>&1; echo ncuf_rc=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_v2 -s 3 -c 1 -o gpurun_out/$TAG/prof_stencil17 python bench.py --workload stencil17 --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu > /dev/null 2>&1; echo ncuf2_rc=$? ;;
probe)
  ./scripts/probe_stride > gpurun_out/$TAG/probe_stride.txt 2>&1; echo probe_rc=$? ;;
variants)
  timeout 600 python scripts/variants.py ${VARIANTS:-write16 stencil17} > gpurun_out/$TAG/variants.txt 2>&1; echo variants_rc=$? ;;
ncustencil)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_v2 -s 2 -c 1 -o gpurun_out/$TAG/prof_stencil17 python bench.py --workload stencil17 --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu > /dev/null 2>&1; echo ncus_rc=$? ;;
part)
  timeout 900 python bench.py --workload part18 --steps 20 --warmup 3 > gpurun_out/$TAG/bench_part18.json 2> gpurun_out/$TAG/bench_part18.err; echo part_rc=$? ;;
e2e)
  timeout 900 python bench.py --no-sweep --no-cpu --steps 50 > gpurun_out/$TAG/bench_e2e.json 2> gpurun_out/$TAG/bench_e2e.err; echo e2e_rc=$? ;;
sysprobe)
  cat /sys/kernel/mm/transparent_hugepage/enabled > gpurun_out/$TAG/probe_sysmem.txt; ./scripts/probe_sysmem >> gpurun_out/$TAG/probe_sysmem.txt 2>&1; ./scripts/probe_sysmem thp >> gpurun_out/$TAG/probe_sysmem.txt 2>&1; echo sys_rc=$? ;;
e2evar)
  timeout 900 python scripts/e2e_variants.py 16 > gpurun_out/$TAG/e2e_variants.txt 2>&1; echo e2evar_rc=$? ;;
profile)
  ./scripts/probe_partial > gpurun_out/$TAG/probe_partial.txt 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/$TAG/probe_partial_ncu.csv ./scripts/probe_partial > /dev/null 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lambda|stencil|l2_flush|fill_hash" -c 60 --csv --log-file gpurun_out/$TAG/launches_write16.csv python bench.py --steps 20 --warmup 3 --no-sweep --no-e2e --no-cpu > /dev/null 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lambda|stencil|l2_flush|fill_hash" -c 40 --csv --log-file gpurun_out/$TAG/launches_stencil17.csv python bench.py --workload stencil17 --steps 10 --warmup 3 --no-sweep --no-e2e --no-cpu > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gasket_write -s 3 -c 1 -o gpurun_out/$TAG/prof_write16 python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_v2 -s 2 -c 1 -o gpurun_out/$TAG/prof_stencil17 python bench.py --workload stencil17 --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu > /dev/null 2>&1
  echo profile_done ;;
nsweep)
  timeout 1500 python bench.py --nsweep --nsweep-out gpurun_out/$TAG/nsweep.csv > gpurun_out/$TAG/nsweep.json 2> gpurun_out/$TAG/nsweep.err; echo nsweep_rc=$? ;;
ab)
  for L in ${ABLIBS:-A B A B}; do echo "== lib$L" >> gpurun_out/$TAG/ab.txt; GASKET_B200_LIB=ab/lib$L.so timeout 600 python scripts/variants.py ${VARIANTS:-stencil17} >> gpurun_out/$TAG/ab.txt 2>&1; done; echo ab_done ;;
fetch)
  for G in def; do A=$G; [ $G = def ] && A=; echo "== granularity $G" >> gpurun_out/$TAG/probe_fetch.txt; ./scripts/probe_fetch $A >> gpurun_out/$TAG/probe_fetch.txt 2>&1
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,dram__bytes_write.sum --csv --log-file gpurun_out/$TAG/probe_fetch_ncu_$G.csv ./scripts/probe_fetch $A > /dev/null 2>&1; done; echo fetch_done ;;
gasket)
  ./scripts/probe_gasket > gpurun_out/$TAG/probe_gasket.txt 2>&1; echo gasket_rc=$?
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/$TAG/probe_gasket_ncu.csv ./scripts/probe_gasket > /dev/null 2>&1 ;;
esac
done
