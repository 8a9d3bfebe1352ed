#!/bin/bash
# ncu --set full captures of the pipelined four-step at 2^20 (k_pipe2) and 2^22 (k_pipe) + DRAM pattern probe.
# The reports are summarised on the box (raw + SASS source CSV) and deleted, to stay under gpurun's 64 MiB.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out/pl
timeout 300 python tools/exp/run_dram2.py > ${O}_dram2.txt 2>&1
for n in ${SIZES:-1048576 4194304}; do
  b=$(( (1<<31) / (8*n) ))
  timeout 300 python tools/ncu_target.py --n $n --batch $b --reps 2 > ${O}_t$n.txt 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pipe -s 1 -c 1 \
    -o /tmp/pl_$n -f python tools/ncu_target.py --n $n --batch $b --reps 2 > ${O}_ncu$n.log 2>&1
  python tools/ncu_summarize.py /tmp/pl_$n.ncu-rep $(( 16 * n * b )) > ${O}_sum$n.md 2>&1
  ncu -i /tmp/pl_$n.ncu-rep --page raw --csv > ${O}_raw$n.csv 2>/dev/null
  ncu -i /tmp/pl_$n.ncu-rep --page source --csv --print-source sass > ${O}_src$n.csv 2>/dev/null
  rm -f /tmp/pl_$n.ncu-rep
done
echo done
