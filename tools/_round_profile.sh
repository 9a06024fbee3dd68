# Round measurement on the GPU box (through gpurun): GPU tests, smoke, the default bench line, the
# per-kernel step profile, the three-stream timeline, the ncu launch list of one step and a
# full-set capture of its tensor-core launches.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-200 gpurun_out/bench.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cut -c1-200 gpurun_out/bench_ref.json
python tools/step_profile.py > gpurun_out/step_profile.txt 2>&1
python tools/timeline.py > gpurun_out/timeline.txt 2>&1
bash tools/_ncu_round.sh
