#!/bin/bash
# r02 call A: toolchain versions, alternate-layout parity of the float-pair pack variants
# (loaded through SDTW_LIB, never overwriting the in-tree library), default GPU suite, bench.
mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
(nvidia-smi; nvcc --version; ptxas --version) > $O/env.txt 2>&1
for v in ptx_o1 ptx_o3 ptx_cl2 ptx_bdp cpp_o1; do
  echo "== $v" >> $O/variants.txt
  SDTW_LIB=$PWD/variants/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=line -k "not config3" 2>&1 | grep -E "passed|failed|Error" | tail -5 >> $O/variants.txt
done
timeout 1500 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -30 > $O/gpu_tests.log
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
SDTW_LIB=$PWD/variants/ptx_o3.so timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > $O/bench_c3_ptx.json 2>&1
