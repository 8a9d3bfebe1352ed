#!/bin/bash
# k_pipe2 (radix-16, 64 KiB tiles) at 2^21 / 2^22 vs k_pipe, with ring size / lag variants; parity first
cd "$(dirname "$0")/../.."
BLOCKFFT_PIPE_IMPL=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "test_pipe and 2097152 or test_pipe and 4194304" 2>&1 | tail -2
echo "== k_pipe (default)"
timeout 120 python tools/time_variants.py --min 21 --max 22 --variants 5 2>&1 | grep -v "^$"
for lag_s in "" "1 2" "1 3" "2 3" "2 4"; do
  set -- $lag_s
  echo "== k_pipe2 LAG=$1 S=$2"
  if [ -n "$1" ]; then export BLOCKFFT_PIPE_LAG=$1 BLOCKFFT_PIPE_S=$2; fi
  BLOCKFFT_PIPE_IMPL=2 timeout 120 python tools/time_variants.py --min 21 --max 22 --variants 5 2>&1 | grep -v "^$"
done
