#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2 | tee gpurun_out/r01m_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/r01m_smoke.log
timeout 600 python bench.py > gpurun_out/r01m_bench_c3.json 2>/dev/null; cut -c1-120 gpurun_out/r01m_bench_c3.json
timeout 600 python bench.py --half --steps 3 > gpurun_out/r01m_bench_c3_half.json 2>/dev/null
timeout 600 python bench.py --config c6_ragged --steps 3 > gpurun_out/r01m_bench_c6_ragged.json 2>/dev/null
timeout 600 python bench.py --config c5_1000 --steps 3 > gpurun_out/r01m_bench_c5_1000.json 2>/dev/null
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
for v in d_bdp d_cl; do cp variants/$v.so paper_2403_06931_b200/libsdtw.so; echo "== $v"; timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=no 2>&1 | tail -1; done
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
