# A/B of two builds on the same box: _ab/old (a worktree of an earlier commit) and the working tree.
cd $GRAFT_REPO_ROOT
for r in 1 2; do
  (cd _ab/old && python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('old', d['ms_per_step'], d['value'])")
  python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('new', d['ms_per_step'], d['value'])"
done
