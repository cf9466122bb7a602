#!/bin/bash
# r02 call H: NCCL/shared-GPU query-shard tests vs the oracle; FADD2 + 2xFFMA cell variant (parity + C3/C2 rate)
O=gpurun_out/r02h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_nccl.py -q -rf --tb=short 2>&1 | tail -20 > $O/nccl_tests.log
SDTW_LIB=$PWD/variants/split.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spec.py -q --tb=line -k "not config3" 2>&1 | tail -5 > $O/split_parity.log
for v in split; do
  SDTW_LIB=$PWD/variants/$v.so timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-e2e > $O/bench_c3_$v.json 2>> $O/bench.err
  SDTW_LIB=$PWD/variants/$v.so timeout 600 python bench.py --config c2 --steps 5 --no-cpu-baseline --no-e2e > $O/bench_c2_$v.json 2>> $O/bench.err
done
timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-e2e > $O/bench_c3_base.json 2>> $O/bench.err
