#!/bin/bash
# Runs on the GPU box: full bench line, the reference arm, then (only after the
# plain command exited 0) the ncu launch list and one full capture per hot kernel.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.csv 2>&1
lscpu > $OUT/lscpu.txt 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo "reference rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD > $OUT/plain.log 2>&1; rc=$?; echo "plain rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
      -k regex:"mark_tma|cap3|writer_warp|writer_kernel|restore" -c 42 --csv \
      --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"${NCU_K:-writer_warp|mark_tma|cap3_count|cap3_emit}" -s ${NCU_S:-16} -c ${NCU_C:-4} \
      -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
