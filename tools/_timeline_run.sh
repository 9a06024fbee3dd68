cd $GRAFT_REPO_ROOT
python tools/timeline.py > gpurun_out/timeline.txt 2>&1
for b in 2 4; do python - <<PY >> gpurun_out/timeline_var.txt 2>&1
import sys; sys.path.insert(0,'.')
from paper_1408_5093_b200 import nets
nets.Net.side_sgd_blocks = $b
import runpy; sys.argv=['x']; print('=== side_sgd_blocks', $b)
runpy.run_path('tools/timeline.py', run_name='__main__')
PY
done
