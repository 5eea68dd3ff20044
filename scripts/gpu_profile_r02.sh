#!/bin/bash
# Runs on the GPU box (one GPU): ncu launch lists and one --set full capture
# per dominant kernel, each only after its plain command exited 0.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; OUT=gpurun_out; mkdir -p $OUT
run() {  # name, ncu filter, skip, count, command...
  local name=$1 k=$2 sk=$3 c=$4; shift 4
  timeout 600 "$@" > $OUT/p_${name}_plain.log 2>&1; local rc=$?; echo "$name plain rc=$rc"
  [ $rc -ne 0 ] && return
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$k" -c 60 --csv \
      --log-file $OUT/p_${name}_launches.csv "$@" > /dev/null 2>&1; echo "$name launches rc=$?"
  [ "$c" -eq 0 ] && return
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${FULLK:-$k}" -s $sk -c $c \
      -o $OUT/p_${name} "$@" > $OUT/p_${name}_ncu.log 2>&1; echo "$name full rc=$?"
}
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --verify-rows 0"
run C2 "mark_tma|cap3|writer_warp" 12 4 $B
run T "writer_warp" 3 1 $B --workload T
run C4 "writer_warp" 3 1 $B --workload C4
run C5 "restore_payload" 18 6 python bench.py --workload C5 --steps 2 --warmup 3 --verify-rows 0
NB=500 SORTED=1 FULLK=train_interval run train "train_|sort_" 0 1 python scripts/bench_train.py
# the reports are too large to travel (gpurun_out <= 64 MiB): summarise here
PROFILE_OUT=$OUT python scripts/make_profiles_r02.py r02 > $OUT/make_profiles.log 2>&1; echo "summary rc=$?"
for f in $OUT/p_*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; done
rm -f $OUT/p_*.ncu-rep
