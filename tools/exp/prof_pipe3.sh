#!/bin/bash
# ncu --set full of k_pipe3 at 2^16 (summarised on the box; report deleted)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out/p3
export BLOCKFFT_PIPE_IMPL=3
n=${N:-65536}; b=$(( (1<<31) / (8*n) ))
timeout 300 python tools/ncu_target.py --n $n --batch $b --reps 2 > ${O}_t.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pipe -s 1 -c 1 \
    -o /tmp/p3 -f python tools/ncu_target.py --n $n --batch $b --reps 2 > ${O}_ncu.log 2>&1
python tools/ncu_summarize.py /tmp/p3.ncu-rep $(( 16 * n * b )) > ${O}_sum.md 2>&1
ncu -i /tmp/p3.ncu-rep --page raw --csv > ${O}_raw.csv 2>/dev/null
ncu -i /tmp/p3.ncu-rep --page source --csv --print-source sass > ${O}_src.csv 2>/dev/null
rm -f /tmp/p3.ncu-rep
