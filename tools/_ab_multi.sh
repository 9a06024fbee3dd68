# A/B/C.. of several builds of the library (graph-replayed step, alternating processes):
#   _ab_multi.sh <reps> <lib.so> [<lib.so> ...]   ("default" = the in-tree build)
cd $GRAFT_REPO_ROOT
R=$1; shift
for i in $(seq $R); do
  for V in "$@"; do
    if [ "$V" = default ]; then L=""; else L=$V; fi
    CAFFE_B200_LIB=$L REPS=1 timeout 300 python tools/sched_sweep.py "skip_update=0" | tail -1 | sed "s|^|$V |"
  done
done
