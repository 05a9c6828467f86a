# parity tests, then walk timings: current library vs scratch/libbdeg_head.so
cd $GRAFT_REPO_ROOT
OUT=gpurun_out; TAG=${1:-wab}
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; rc=$?; echo "pytest rc $rc"; tail -2 $OUT/pytest_gpu_$TAG.log
for i in 1 2; do
  for lib in paper_1501_02237_b200/libbdeg.so scratch/libbdeg_head.so; do
    BDEG_LIB=$lib timeout 300 python tools/walk_runs.py w44,w36,w45,w37 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$lib', d['wl'], '%.3f s' % d['walk_s'], d['degree'])"
  done
done
