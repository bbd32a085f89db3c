cd $GRAFT_REPO_ROOT
for dbg in 0 1 2 4 6 7; do echo "debug $dbg" >> gpurun_out/c16_dbg.log; DGNN_UMMA_DEBUG=$dbg python scripts/kernel_bench.py --only cell_fwd_gru,cell_bwd_gru --n 4000000 --prof 2>&1 | grep -A2 "row_gemm" >> gpurun_out/c16_dbg.log; done
