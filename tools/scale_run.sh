#!/bin/bash
# bench.py at N = 1, 2, 4 GPUs (torchrun, one rank per GPU) + the reference arm at N = 4 +
# the host streamer with 4 concurrent GPUs.  Run under gpurun --gpus 4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/sc
timeout 600 python bench.py --steps 20 --warmup 5 > ${O}_n1.txt 2>&1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + n)) bench.py --gpus $n --steps 20 --warmup 5 > ${O}_n$n.txt 2>&1
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29510 bench.py --impl reference --gpus 4 --steps 2 --warmup 3 > ${O}_ref4.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29511 tools/stream_bench.py --buf-gib 4 --passes 4 --file-gib 8 > ${O}_stream4.txt 2>&1
echo done
