#!/bin/bash
# One iteration of sliced-K1 work on the GPU box: accuracy + timing +
# determinism (tools/diag/sliced_check.py), the sliced pytest file, the CTA-0
# timeline. usage: tools/sliced_iter.sh TAG [extra pytest files...]
TAG=${1:-it}; shift
O=gpurun_out; mkdir -p $O
timeout 600 python tools/diag/sliced_check.py > $O/${TAG}_check.txt 2>&1; echo check rc=$?
timeout 900 python -m pytest -x -q tests/test_spmm_sliced_gpu.py "$@" > $O/${TAG}_pytest.txt 2>&1; echo pytest rc=$?
timeout 300 python tools/diag/sliced_trace.py > $O/${TAG}_trace.txt 2>&1; echo trace rc=$?
tail -3 $O/${TAG}_pytest.txt; cat $O/${TAG}_check.txt
