#!/bin/bash
# ring size / lag at 2^21, 2^22 (k_pipe): smaller rings stay in L2
cd "$(dirname "$0")/../.."
for lag_s in "1 2" "1 3" "2 3" "2 4" "3 5"; do
  set -- $lag_s
  echo "== LAG=$1 S=$2"
  BLOCKFFT_PIPE_LAG=$1 BLOCKFFT_PIPE_S=$2 timeout 120 python tools/time_variants.py --min 21 --max 22 --variants 5 2>&1 | grep -v "^$"
done
