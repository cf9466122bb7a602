#!/bin/bash
# r02 call AS: the two-segment split tests and the suites that touch the speculative plan
O=gpurun_out/r02as; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_spec.py tests/test_gpu_start_ckpt.py tests/test_gpu_tail_skip.py tests/test_gpu_ragged.py tests/test_gpu_half.py tests/test_gpu_q8.py tests/test_gpu_refsplit.py -q -x -rf --tb=short 2>&1 | tail -15 > $O/tests.log
cat $O/tests.log
