#!/bin/bash
# Builder-side scaling evidence on one box with up to 4 GPUs (the driver's SCALE run needs 8):
# config 2 (weak) and config 3 (strong) at N = 1, 2, 4; the 1 TiB host stream at G = 1, 2, 4;
# one record over G GPUs (fft_dplan) at 2^30 and 2^32.  Output: gpurun_out/scale/*.
mkdir -p gpurun_out/scale
for cfg in 2 3; do
  python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/scale/c${cfg}_n1.txt 2>&1
  for N in 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 2953$N bench.py --gpus $N --config $cfg --steps 20 --warmup 5 --e2e-steps 3 > gpurun_out/scale/c${cfg}_n$N.txt 2>&1
  done
done
timeout 1200 python tools/stream_tib.py --gpus 1,2,4 --tib 1.0 --json gpurun_out/scale/tib.json > gpurun_out/scale/tib.txt 2>&1
python tools/dplan_bench.py --log2n 30 --gpus 1,2,4 --json gpurun_out/scale/dplan30.json > gpurun_out/scale/dplan30.txt 2>&1
python tools/dplan_bench.py --log2n 32 --gpus 1,2,4 --json gpurun_out/scale/dplan32.json > gpurun_out/scale/dplan32.txt 2>&1
for f in gpurun_out/scale/c*_n*.txt; do echo "$f: $(grep -o '"value": [0-9.e+]*' $f | head -1) $(grep -o '"frac": [0-9.]*' $f | head -1)"; done
cat gpurun_out/scale/dplan30.txt gpurun_out/scale/dplan32.txt
