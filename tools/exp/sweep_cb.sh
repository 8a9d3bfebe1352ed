#!/bin/bash
# k_pipe2 claim batching A/B (BLOCKFFT_PIPE_CB = 1 / 2) at 2^15..2^18, plus the default choice 2^13..2^22 + parity
cd "$(dirname "$0")/../.."
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "pipe or auto" 2>&1 | tail -2
BLOCKFFT_PIPE_CB=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "pipe" 2>&1 | tail -2
for cb in 1 2; do
  echo "== CB=$cb"
  BLOCKFFT_PIPE_CB=$cb timeout 240 python tools/time_variants.py --min 15 --max 18 --variants 5 2>&1 | grep -v "^$"
done
echo "== default"
timeout 300 python tools/time_variants.py --min 13 --max 22 --variants 0 2>&1 | grep -v "^$"
