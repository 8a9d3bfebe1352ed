#!/bin/bash
# 2^14 as a 2-CTA cluster (64 KiB per CTA): every cluster implementation vs the defaults
cd "$(dirname "$0")/../.."
BLOCKFFT_CLUSTER_SIZE=2 BLOCKFFT_CLUSTER_IMPL=1 timeout 200 python -m pytest tests/test_gpu_parity.py -q -x -k "test_cluster and 16384" 2>&1 | tail -1
for cfg in "0 0" "1 2" "1 3" "2 0"; do
  set -- $cfg
  echo "== impl=$1 minb=$2 C=2"
  BLOCKFFT_CLUSTER_SIZE=2 BLOCKFFT_CLUSTER_IMPL=$1 BLOCKFFT_CLUSTER_MINB=$2 timeout 120 python tools/time_variants.py --min 14 --max 14 --variants 2 2>&1 | grep -v "^$"
done
echo "== defaults"
timeout 120 python tools/time_variants.py --min 14 --max 14 --variants 1,2,5 2>&1 | grep -v "^$"
