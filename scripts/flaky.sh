#!/bin/bash
mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "test_config1_bit_exact_all_schedules" 2>&1 | tail -3; done > gpurun_out/flaky_new.log
cp paper_2403_06931_b200/libsdtw.so /tmp/new.so; cp variants/base.so paper_2403_06931_b200/libsdtw.so
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "test_config1_bit_exact_all_schedules" 2>&1 | tail -3; done > gpurun_out/flaky_base.log
cp /tmp/new.so paper_2403_06931_b200/libsdtw.so
echo NEW; cat gpurun_out/flaky_new.log; echo BASE; cat gpurun_out/flaky_base.log
