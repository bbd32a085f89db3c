cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests8.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests8.log
