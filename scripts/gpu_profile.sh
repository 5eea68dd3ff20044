#!/bin/bash
# Runs on the GPU box: plain bench, then the ncu launch list and a full capture of the top kernels.
set -u
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
$CMD > $OUT/plain.log 2>&1; rc=$?; echo "plain rc=$rc"
if [ $rc -eq 0 ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:"writer_kernel|mark_kernel|capture_write" \
      -s 7 -c 3 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
