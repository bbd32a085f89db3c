cd $GRAFT_REPO_ROOT
KB="python scripts/kernel_bench.py --n 4000000 --iters 10"
for cfg in "" "DGNN_DELTA_MINB=3" "DGNN_DELTA_MINB=4" "DGNN_L2_PERSIST_MB=200" "DGNN_L2_PERSIST_MB=200 DGNN_DELTA_MINB=3"; do
  echo "== $cfg" >> gpurun_out/kb2.log
  env $cfg timeout 300 $KB --only agg_delta_feat >> gpurun_out/kb2.log 2>&1
done
timeout 300 $KB --only agg_scratch128,agg_scratch64,agg_backward64,agg_delta >> gpurun_out/kb2.log 2>&1
for cfg in "" "DGNN_L2_PERSIST_MB=200"; do
  env $cfg timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_agg_delta_v4 -c 2 python scripts/kernel_bench.py --only agg_delta_feat --n 4000000 --iters 1 >> gpurun_out/ncu2.log 2>&1
done
python - <<'PY' >> gpurun_out/kb2.log 2>&1
import torch
p = torch.cuda.get_device_properties(0)
print("l2", p.L2_cache_size, "persist max", getattr(p, "persisting_l2_cache_max_size", None))
PY
