#!/bin/bash
# TMA L2 promotion of the A-tile tensor map (0 none .. 3 256 B), pipelined sizes
cd "$(dirname "$0")/../.."
for p in 3 2 0; do
  echo "== promo=$p"
  BLOCKFFT_TMAP_PROMO=$p timeout 200 python tools/time_variants.py --min 14 --max 22 --variants 5 2>&1 | grep -v "^$"
done
