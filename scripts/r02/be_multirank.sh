#!/bin/bash
# r02 call BE (re-run on the final library): the bench's multi-rank path on the one GPU (2 ranks, gloo records, shared GPU) --
# functional check of sharding / barrier / max-over-ranks / JSON line; plus the NCCL world-1 line
O=gpurun_out/r02be; mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
   bench.py --gpus 2 --steps 2 --warmup 3 --backend gloo --config c2 > $O/bench_2rank_gloo_c2.json 2> $O/bench_2rank.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 \
   bench.py --gpus 1 --steps 2 --warmup 3 --config c2 > $O/bench_1rank_nccl_c2.json 2> $O/bench_1rank.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 1 --steps 2 --warmup 3 > $O/bench_1rank_nccl_c3.json 2> $O/bench_1rank_c3.err
cat $O/*.json; for f in $O/*.err; do tail -n 3 $f; done
