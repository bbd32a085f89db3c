cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests3.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests3.log
KB="python scripts/kernel_bench.py --n 4000000 --iters 10"
for cfg in "DGNN_DELTA_ST_HINT=0" "DGNN_DELTA_ST_HINT=1"; do
  echo "== $cfg" >> gpurun_out/kb3.log
  env $cfg timeout 300 $KB --only agg_delta_feat >> gpurun_out/kb3.log 2>&1
  env $cfg timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_agg_delta_v4 -c 1 python scripts/kernel_bench.py --only agg_delta_feat --n 4000000 --iters 1 >> gpurun_out/ncu3.log 2>&1
done
timeout 300 $KB --only cell_bwd_gru --prof >> gpurun_out/kb3.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err
