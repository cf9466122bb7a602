#!/bin/bash
# r02 call Q: the float-pair pack defect -- which parity cases fail for the inline-PTX pack at
# ptxas -O3 / -O1 / -O0, and the C++ pack at -O0 (same PTX semantics; -O0 = no ptxas optimisation)
O=gpurun_out/r02q; mkdir -p $O
for v in ptx_o3 ptx_o1 ptx_o0 cpp_o0; do
  echo "== $v" >> $O/variants.txt
  SDTW_LIB=$PWD/variants/$v.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rf --tb=no -p no:cacheprovider \
     -k "config1_bit_exact or ragged_shapes or quantised or config5_shape" 2>&1 | grep -E "^FAILED|passed|failed" >> $O/variants.txt
done
