cd $GRAFT_REPO_ROOT
(cd _ab/old && python tools/step_profile.py > ../../gpurun_out/sp_old.txt 2>&1)
python tools/step_profile.py > gpurun_out/sp_new.txt 2>&1
(cd _ab/old && python tools/timeline.py > ../../gpurun_out/tl_old.txt 2>&1)
python tools/timeline.py > gpurun_out/tl_new.txt 2>&1
