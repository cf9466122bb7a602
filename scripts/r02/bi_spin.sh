#!/bin/bash
# r02 call BI: flow-control poll sleep (SDTW_SPIN_NS) -- the wait loop issued 6.8 % of the C3 launch's
# warp instructions at 256 ns (r02bd source page); variants built into variants/ (SDTW_LIB)
O=gpurun_out/r02bi; mkdir -p $O
for lib in "" variants/spin512.so variants/spin1024.so variants/spin2048.so; do
  tag=${lib:-default}
  SDTW_LIB=$lib Z=512 N=2000 M=10000000 CONFIGS='[{}, {}]' timeout 600 python scripts/sweep.py | sed "s#^#{\"lib\": \"$tag\", \"w\": \"c3\", \"r\": #; s/$/}/" >> $O/spin.jsonl 2>&1
  SDTW_LIB=$lib Z=512 N=2000 M=100000 CONFIGS='[{}, {}]' timeout 600 python scripts/sweep.py | sed "s#^#{\"lib\": \"$tag\", \"w\": \"c2\", \"r\": #; s/$/}/" >> $O/spin.jsonl 2>&1
  SDTW_LIB=$lib TRACE=1 Z=512 N=1000 M=1000000 CONFIGS='[{}, {}]' timeout 600 python scripts/sweep.py | sed "s#^#{\"lib\": \"$tag\", \"w\": \"c5_1000\", \"r\": #; s/$/}/" >> $O/spin.jsonl 2>&1
  SDTW_LIB=$lib TRACE=1 Z=512 N=8000 M=1000000 CONFIGS='[{}]' timeout 600 python scripts/sweep.py | sed "s#^#{\"lib\": \"$tag\", \"w\": \"c5_8000\", \"r\": #; s/$/}/" >> $O/spin.jsonl 2>&1
done
cat $O/spin.jsonl
