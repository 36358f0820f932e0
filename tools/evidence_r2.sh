#!/bin/bash
# Round-2 evidence pass on one B200 (gpurun): GPU suite, bench (both arms),
# launch list, DRAM traffic of one config-2 SpMM call, --set full of the
# sliced K1, CTA-0 timeline. Every ncu pass runs after its command exited 0.
# usage: tools/evidence_r2.sh TAG [skip-tests]
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${TAG}_smi.txt
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.txt 2>&1; echo pytest rc=$?
fi
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_ref.json 2> $O/${TAG}_ref.err; echo ref rc=$?
timeout 900 python tools/diag/sliced_prof.py 16 auto > /dev/null 2>&1 && \
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    python tools/diag/sliced_prof.py 16 auto > $O/${TAG}_traffic_m16.csv 2>&1; echo traffic rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cfg4 --no-cpu-baseline > $O/${TAG}_ncu_bench.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_sliced -s 1 -c 1 -o $O/${TAG}_sliced_full \
  python tools/diag/sliced_prof.py 16 sliced > $O/${TAG}_sliced_full.log 2>&1; echo ncu2 rc=$?
timeout 600 python tools/diag/sliced_trace.py > $O/${TAG}_sliced_trace.txt 2>&1; echo trace rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fom_fast -s 2 -c 1 -o $O/${TAG}_fom_full \
  python tools/prof_cfg4_iter.py 8 > $O/${TAG}_fom_full.log 2>&1; echo ncu3 rc=$?
