#!/bin/bash
# A/B of k_pipe2 compute-group configurations (BLOCKFFT_PIPE_GRP = 1, 2, 4) at 2^15..2^20
cd "$(dirname "$0")/../.."
for g in 1 2 4; do
  echo "== GRP=$g"
  BLOCKFFT_PIPE_GRP=$g timeout 300 python tools/time_variants.py --min ${MINL:-15} --max ${MAXL:-20} --variants 5 2>&1 | grep -v "^$"
done
