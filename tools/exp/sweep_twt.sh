#!/bin/bash
# k_pipe2: four-step twiddles from a full [k1][n2] table (TWT=1) vs the two-level lookup + tree (TWT=0), 2^14..2^16
cd "$(dirname "$0")/../.."
BLOCKFFT_PIPE_TWT=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "test_pipe and (16384 or 32768 or 65536 or 131072 or 262144)" 2>&1 | tail -1
for r in 1; do for t in 0 1; do
  echo "== TWT=$t (repeat $r)"
  BLOCKFFT_PIPE_TWT=$t timeout 200 python tools/time_variants.py --min 14 --max 18 --variants 5 2>&1 | grep -v "^$"
done; done
