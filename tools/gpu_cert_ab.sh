# certificate pruning: parity tests, then C5 / W26 benches with and without it
cd $GRAFT_REPO_ROOT
OUT=gpurun_out; TAG=${1:-cert}
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?"; tail -3 $OUT/pytest_gpu_$TAG.log
python bench.py --no-cpu-baseline > $OUT/bench_c5_$TAG.log 2>&1; tail -1 $OUT/bench_c5_$TAG.log | cut -c1-250
BDEG_NO_CERT=1 python bench.py --no-cpu-baseline > $OUT/bench_c5_nocert_$TAG.log 2>&1; tail -1 $OUT/bench_c5_nocert_$TAG.log | cut -c1-250
python bench.py --workload w26 --steps 3 --no-cpu-baseline > $OUT/bench_w26_$TAG.log 2>&1; tail -1 $OUT/bench_w26_$TAG.log | cut -c1-250
