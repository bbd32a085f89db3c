cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_cache_policies.py -x -q > gpurun_out/gputests6.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests6.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_row_gemm -c 1 -o gpurun_out/ncu_rowgemm_gru python scripts/kernel_bench.py --n 4000000 --iters 1 --only cell_fwd_gru > gpurun_out/ncu6.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_agg_delta_v4 -c 1 -o gpurun_out/ncu_delta_v5 python scripts/kernel_bench.py --n 4000000 --iters 1 --only agg_delta_feat >> gpurun_out/ncu6.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wgrad -c 1 -o gpurun_out/ncu_wgrad_v2 python scripts/kernel_bench.py --n 4000000 --iters 1 --only cell_bwd_gru >> gpurun_out/ncu6.log 2>&1
