#!/bin/bash
# A/B sweep of the cluster kernel implementations at 2^16 (and neighbours).
cd "$(dirname "$0")/.."
run() { echo "== $*"; env "$@" timeout 120 python tools/time_variants.py --min ${MINL:-16} --max ${MAXL:-16} --gib 2 --variants 2 2>&1 | grep -v "^$"; }
for impl in 0 1; do
  if [ $impl = 0 ]; then
    for xch in 0 1; do for c in 8 16; do run BLOCKFFT_CLUSTER_IMPL=0 BLOCKFFT_CLUSTER_XCH=$xch BLOCKFFT_CLUSTER_SIZE=$c; done; done
  else
    for c in 8 16; do for mb in 1 2 3 4; do run BLOCKFFT_CLUSTER_IMPL=1 BLOCKFFT_CLUSTER_SIZE=$c BLOCKFFT_CLUSTER_MINB=$mb; done; done
  fi
done
