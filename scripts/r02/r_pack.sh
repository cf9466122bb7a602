#!/bin/bash
# r02 call R: the float-pair pack reproducer under each build
O=gpurun_out/r02r; mkdir -p $O
for v in ptx_o3 ptx_o1 ptx_o0 cpp_o0; do
  SDTW_LIB=$PWD/variants/$v.so timeout 300 python scripts/pack_repro.py >> $O/repro.txt 2>&1
done
timeout 300 python scripts/pack_repro.py >> $O/repro.txt 2>&1
