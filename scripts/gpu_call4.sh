cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_khop.py tests/test_dataset_io.py -x -q > gpurun_out/gputests4.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests4.log
timeout 600 python scripts/dataset_bench.py > gpurun_out/dataset_bench_c1.json 2> gpurun_out/dataset_bench.err
timeout 900 python scripts/dataset_bench.py --n 1000000 --deg 20 --dim 128 --T 4 --edge 0.02 --feat 0.0 --reps 2 > gpurun_out/dataset_bench_c3.json 2>> gpurun_out/dataset_bench.err
