#!/bin/bash
# r02 call C: start-index select on the FMA pipe (parity + C5 benches); C=4 chains at 16 warps/SM
O=gpurun_out/r02c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spec.py tests/test_gpu_path.py tests/test_gpu_ragged.py -q -x 2>&1 | tail -3 > $O/tests.log
for c in c5_500 c5_1000 c5_4000 c5_8000; do
  timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2>> $O/bench.err
done
CFG='[{}, {"OPT_PACKED": 2, "OPT_SEGMENT_W": 28, "OPT_LANES": 4}]'
M=10000000 CONFIGS="$CFG" timeout 600 python scripts/sweep.py > $O/sweep_default_lib.jsonl 2>&1
CFG='[{}, {"OPT_PACKED": 2, "OPT_SEGMENT_W": 28, "OPT_LANES": 4}, {"OPT_PACKED": 2, "OPT_SEGMENT_W": 28, "OPT_LANES": 2}, {"OPT_PACKED": 2, "OPT_SEGMENT_W": 28, "OPT_LANES": 4, "OPT_CHUNK": 64}]'
SDTW_LIB=$PWD/variants/c4b4.so M=10000000 CONFIGS="$CFG" timeout 600 python scripts/sweep.py > $O/sweep_c4b4.jsonl 2>&1
