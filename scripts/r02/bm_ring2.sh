#!/bin/bash
# r02 call BM: 2-warp plans shallow their inter-warp rings up to 8 resident CTAs -- tests and config-5 lines
O=gpurun_out/r02bm; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_start_ckpt.py tests/test_gpu_spec.py tests/test_gpu_parity.py tests/test_gpu_path.py tests/test_gpu_tail_skip.py "tests/test_gpu_fullsize.py::test_config5_start_index_vs_full_reference_oracle" -q -x -rf --tb=short 2>&1 | tail -15 > $O/tests.log
for c in c5_500 c5_1000; do timeout 900 python bench.py --config $c --steps 5 --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err; done
timeout 900 python bench.py --config c5_1000 --steps 5 --no-cpu-baseline --path > $O/bench_c5_1000_path.json 2>> $O/bench.err
cat $O/tests.log; tail -3 $O/bench.err
