cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu -k "not walk" > gpurun_out/pytest_ab4.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_ab4.log
LIBS="scratch/libbdeg_head.so" bash tools/gpu_ab3.sh
