cd $GRAFT_REPO_ROOT
OUT=gpurun_out; TAG=${1:-chk}
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?"; tail -2 $OUT/pytest_gpu_$TAG.log
python bench.py --impl reference --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-160
for lib in paper_1501_02237_b200/libbdeg.so scratch/libbdeg_head.so; do
  BDEG_LIB=$lib timeout 300 python tools/walk_runs.py c5,w36 2>&1 | grep '^{' | cut -c1-120
done
