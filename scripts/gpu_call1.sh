cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 300 python scripts/kernel_bench.py --only agg_delta_feat,cell_bwd_gru --n 4000000 --iters 5 --prof > gpurun_out/kb.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_agg_delta_v4 -c 1 -o gpurun_out/ncu_delta python scripts/kernel_bench.py --only agg_delta_feat --n 4000000 --iters 1 > gpurun_out/ncu_delta.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wgrad -c 1 -o gpurun_out/ncu_wgrad python scripts/kernel_bench.py --only cell_bwd_gru --n 4000000 --iters 1 > gpurun_out/ncu_wgrad.log 2>&1
echo done
