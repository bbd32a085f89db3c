cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputests10.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests10.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/bench10_n2.json 2> gpurun_out/bench10_n2.err
