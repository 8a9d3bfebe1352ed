#!/bin/bash
# bench.py --config 3 (16 GiB of 2^20-point records per GPU) at N = 1, 2, 4 GPUs.  Run under gpurun --gpus 4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/sc3
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 --e2e-steps 2 > ${O}_n1.txt 2>&1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29520 + n)) bench.py --config 3 --gpus $n --steps 10 --warmup 3 --e2e-steps 2 > ${O}_n$n.txt 2>&1
done
echo done
