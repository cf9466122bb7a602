#!/bin/bash
# r02 call J: full GPU suite after the dp2 refactor / q8 / speculative-fixup change; worst-case bench
O=gpurun_out/r02j; mkdir -p $O
timeout 2000 python -m pytest tests -m gpu -q -rf --tb=short 2>&1 | tail -30 > $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py --config c3_straddle --steps 3 --no-cpu-baseline --no-e2e > $O/bench_c3_straddle.json 2>> $O/bench.err
SDTW_LIB=$PWD/variants/fixseq.so timeout 600 python bench.py --config c3_straddle --steps 3 --no-cpu-baseline --no-e2e > $O/bench_c3_straddle_fixseq.json 2>> $O/bench.err
timeout 600 python bench.py --config c3 --steps 3 --no-cpu-baseline --no-e2e > $O/bench_c3.json 2>> $O/bench.err
