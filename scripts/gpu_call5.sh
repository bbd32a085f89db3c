cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests5.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests5.log
for cfg in "DGNN_GRU_SPLIT=0" "DGNN_GRU_SPLIT=1"; do
  echo "== $cfg" >> gpurun_out/kb5.log
  env $cfg timeout 300 python scripts/kernel_bench.py --n 4000000 --iters 10 --only cell_fwd_gru >> gpurun_out/kb5.log 2>&1
  env $cfg timeout 300 python scripts/kernel_bench.py --n 4000000 --d 64 --iters 10 --only cell_fwd_gru >> gpurun_out/kb5.log 2>&1
done
timeout 1200 python bench.py > gpurun_out/bench5.json 2> gpurun_out/bench5.err
