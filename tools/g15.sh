#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python tools/rank_share.py > gpurun_out/g15_rank_share.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gather --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g15_gather_p2p.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gather --gather-mode nccl --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g15_gather_nccl.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g15_ref.log 2>&1
