cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests9.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests9.log
P8=$GRAFT_REPO_ROOT/build/p8/_dgnn_b200_p8.so
DGNN_LIB_PATH=$P8 timeout 600 python -m pytest tests/test_gpu_parity.py -k "cell or tensor_core" -x -q > gpurun_out/gputests9_p8.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests9_p8.log
for lib in "" "$P8"; do
  echo "== lib $lib" >> gpurun_out/kb9.log
  DGNN_LIB_PATH=$lib timeout 300 python scripts/kernel_bench.py --n 4000000 --iters 10 --only cell_fwd_gru,cell_fwd_lstm >> gpurun_out/kb9.log 2>&1
  DGNN_LIB_PATH=$lib timeout 300 python scripts/kernel_bench.py --n 4000000 --iters 10 --only cell_bwd_gru --prof >> gpurun_out/kb9.log 2>&1
done
