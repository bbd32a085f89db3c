cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests11.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests11.log
timeout 1500 python bench.py > gpurun_out/bench11.json 2> gpurun_out/bench11.err
