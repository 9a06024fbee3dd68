# A/B of two builds of the library (graph-replayed step, alternating processes): _ab_lib.sh <variant.so> [reps]
cd $GRAFT_REPO_ROOT
V=$1; R=${2:-3}
for i in $(seq $R); do
  REPS=1 timeout 300 python tools/sched_sweep.py "skip_update=0" | tail -1 | sed "s/^/base    /"
  CAFFE_B200_LIB=$V REPS=1 timeout 300 python tools/sched_sweep.py "skip_update=0" | tail -1 | sed "s/^/variant /"
done
