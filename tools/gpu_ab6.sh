cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu -k "walk or table3 or cells" > gpurun_out/pytest_ab6.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_ab6.log
for i in 1 2; do
  for lib in paper_1501_02237_b200/libbdeg.so scratch/libbdeg_prev.so; do
    BDEG_LIB=$lib timeout 300 python tools/walk_runs.py w36,w45,w37 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$lib', d['wl'], '%.3f s' % d['walk_s'], d['degree'])"
  done
done
