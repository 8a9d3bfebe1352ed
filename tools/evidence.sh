#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): GPU tests, the bench line,
# its ncu launch list, one ncu --set full capture of the dominant kernel at the
# bench size, and the variant sweep.  Everything lands in gpurun_out/ev_*.
# Each ncu pass runs only after the same command exited 0 without ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/ev
timeout 1200 python -m pytest tests -q -m gpu -x > ${O}_pytest.txt 2>&1; echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > ${O}_bench.txt 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file ${O}_launches.csv python bench.py --steps 2 --warmup 3 > ${O}_bench_ncu.log 2>&1
timeout 300 python tools/ncu_target.py --n 65536 --batch 8192 --reps 2 > ${O}_target.txt 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pipe -s 1 -c 1 \
    -o /tmp/ev_pipe2 -f python tools/ncu_target.py --n 65536 --batch 8192 --reps 2 > ${O}_ncu_full.log 2>&1
python tools/ncu_summarize.py /tmp/ev_pipe2.ncu-rep 8589934592 > ${O}_ncu_sum.md 2>&1   # summarised here:
rm -f /tmp/ev_pipe2.ncu-rep                                                               # gpurun_out <= 64 MiB
timeout 900 python tools/time_variants.py --min 7 --max 22 --variants 0,1,2,5 --json ${O}_sweep.json > ${O}_sweep.txt 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > ${O}_ref.txt 2>&1
echo done
