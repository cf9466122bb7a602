#!/bin/bash
# r02 call BG: tail skip with cluster rings and 4 / 1 chains per lane
O=gpurun_out/r02bg; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_tail_skip.py -q -rf --tb=short 2>&1 | tail -15 > $O/tests.log
cat $O/tests.log
