mkdir -p gpurun_out
export CONFIGS='[{"OPT_PACKED":1,"OPT_SEGMENT_W":30,"OPT_LANES":4},{"OPT_PACKED":1,"OPT_SEGMENT_W":30,"OPT_LANES":4,"OPT_WORKERS":4}]'
timeout 300 python scripts/sweep.py > gpurun_out/ab_alt1.jsonl 2>&1
cp paper_2403_06931_b200/libsdtw.so variants/alt1_backup.so; cp variants/libsdtw_alt0.so paper_2403_06931_b200/libsdtw.so
timeout 300 python scripts/sweep.py > gpurun_out/ab_alt0.jsonl 2>&1
cp variants/alt1_backup.so paper_2403_06931_b200/libsdtw.so
timeout 600 python -m pytest tests -m gpu -x -q --timeout 400 > gpurun_out/pytest_alt1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp -s 1 -c 1 -o gpurun_out/alt1_dp python scripts/prof_one.py > gpurun_out/alt1_ncu.log 2>&1
cat gpurun_out/ab_alt1.jsonl gpurun_out/ab_alt0.jsonl; tail -3 gpurun_out/pytest_alt1.log; tail -3 gpurun_out/alt1_ncu.log
