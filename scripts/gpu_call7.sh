cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_cache_policies.py -x -q > gpurun_out/gputests7.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests7.log
timeout 900 python scripts/khop_bench.py > gpurun_out/khop_bench.json 2> gpurun_out/khop_bench.err
timeout 900 python scripts/khop_bench.py --n 1000000 --seeds 10000 > gpurun_out/khop_bench_1m.json 2>> gpurun_out/khop_bench.err
