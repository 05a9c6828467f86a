cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_ab5.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_ab5.log
LIBS="scratch/libbdeg_head.so" bash tools/gpu_ab3.sh
for wl in w24 w25; do for lib in paper_1501_02237_b200/libbdeg.so scratch/libbdeg_head.so; do
  echo "$lib $wl $(BDEG_LIB=$lib python bench.py --workload $wl --steps 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")"; done; done
