#!/bin/bash
# One GPU pass: parity tests, benches, launch list and a full ncu capture of the top kernel.
# Usage (under gpurun): bash tools/runs/gpu_round.sh <tag> [full]
TAG=${1:-dev}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?"; tail -3 $OUT/pytest_gpu_$TAG.log
python bench.py > $OUT/bench_c5_$TAG.log 2>&1; tail -1 $OUT/bench_c5_$TAG.log | cut -c1-400
python bench.py --workload w26 --steps 3 --no-cpu-baseline > $OUT/bench_w26_$TAG.log 2>&1; tail -1 $OUT/bench_w26_$TAG.log | cut -c1-300
if [ "$2" == "full" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 6 -c 1 -o $OUT/prof_c5_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 6 -c 1 -o $OUT/prof_w24_$TAG python bench.py --workload w24 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
fi
ls $OUT
