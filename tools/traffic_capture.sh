#!/bin/bash
# DRAM bytes per config-2 SpMM call (m = 16, the default kernel), summed over
# the call's kernels: ncu --metrics on the 4th..6th calls of tools/diag/sliced_prof.py.
set -e
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    python tools/diag/sliced_prof.py 16 auto > gpurun_out/traffic_m16.csv 2>&1
