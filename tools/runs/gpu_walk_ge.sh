cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -x -q -m gpu -k "walk" > gpurun_out/pytest_walk_s3.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_walk_s3.log
export BDEG_DEBUG=1
BDEG_WALK_CAP0=1024 timeout 300 python tools/walk_runs.py w45,w37 > gpurun_out/walk_evict_s3.log 2>&1; tail -4 gpurun_out/walk_evict_s3.log
BDEG_DEBUG_LEVELS=1 timeout 1500 python tools/walk_runs.py w46 > gpurun_out/walk_w46_s3.log 2>&1; echo "w46 rc $?"; tail -4 gpurun_out/walk_w46_s3.log
