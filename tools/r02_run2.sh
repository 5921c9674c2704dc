mkdir -p gpurun_out/r2
timeout -s KILL 900 python -m pytest tests/test_gpu_sharded.py -x -q -p no:cacheprovider > gpurun_out/r2/pytest_sharded.txt 2>&1; tail -15 gpurun_out/r2/pytest_sharded.txt
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/pytest_gpu.txt 2>&1; tail -3 gpurun_out/r2/pytest_gpu.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2/bench_c3.json 2> gpurun_out/r2/bench_c3.err; tail -c 600 gpurun_out/r2/bench_c3.json; tail -3 gpurun_out/r2/bench_c3.err
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2/bench_c4.json 2> gpurun_out/r2/bench_c4.err; tail -c 1500 gpurun_out/r2/bench_c4.json; tail -3 gpurun_out/r2/bench_c4.err
