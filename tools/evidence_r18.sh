set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r18_smi.txt
python bench.py > gpurun_out/bench18.json 2> gpurun_out/bench18.err; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref18.json 2> gpurun_out/ref18.err; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r18_launches.csv python bench.py --steps 3 --warmup 3 --no-cfg4 --no-cpu-baseline > gpurun_out/r18_ncu_bench.log 2>&1; echo ncu1 rc=$?
ncu --set full --import-source on --clock-control none -k regex:spmm_ws -s 2 -c 1 -o gpurun_out/r18_k1_full python tools/prof_spmm.py --m 16 --reps 3 > gpurun_out/r18_k1_full.log 2>&1; echo ncu2 rc=$?
ncu --set full --import-source on --clock-control none -k regex:spmm_ws -s 2 -c 1 -o gpurun_out/r18_k1sp_full python tools/prof_spmm.py --m 8 --reps 3 > gpurun_out/r18_k1sp_full.log 2>&1; echo ncu3 rc=$?
