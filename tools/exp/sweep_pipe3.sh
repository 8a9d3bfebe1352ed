#!/bin/bash
# k_pipe3 (compute groups, early stage release): parity at 2^15..2^20 then A/B timing of its
# (stages, groups) configurations against k_pipe2
cd "$(dirname "$0")/../.."
BLOCKFFT_PIPE_IMPL=3 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "pipe" 2>&1 | tail -3
for c in ${CFGS:-0 1 2 3 4}; do
  echo "== k_pipe3 cfg=$c"
  BLOCKFFT_PIPE_IMPL=3 BLOCKFFT_PIPE3_CFG=$c timeout 240 python tools/time_variants.py --min ${MINL:-15} --max ${MAXL:-20} --variants 5 2>&1 | grep -v "^$"
done
echo "== k_pipe2"
timeout 240 python tools/time_variants.py --min ${MINL:-15} --max ${MAXL:-20} --variants 5 2>&1 | grep -v "^$"
