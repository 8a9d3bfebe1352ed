#!/bin/bash
# k_pipe2 radix-32: direct constant-table twiddles (TWD=1) vs the multiply tree (TWD=0), 2^14..2^18
cd "$(dirname "$0")/../.."
BLOCKFFT_PIPE_TWD=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "pipe" 2>&1 | tail -1
for r in 1 2; do for t in 0 1; do
  echo "== TWD=$t (repeat $r)"
  BLOCKFFT_PIPE_TWD=$t timeout 200 python tools/time_variants.py --min 14 --max 18 --variants 5 2>&1 | grep -v "^$"
done; done
