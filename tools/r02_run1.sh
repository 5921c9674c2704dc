mkdir -p gpurun_out/r1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1/smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r1/pytest_gpu.txt 2>&1; tail -3 gpurun_out/r1/pytest_gpu.txt
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/r1/bench_c3.json 2> gpurun_out/r1/bench_c3.err; tail -c 3000 gpurun_out/r1/bench_c3.json
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu > gpurun_out/r1/bench_c2.json 2> gpurun_out/r1/bench_c2.err; tail -c 1500 gpurun_out/r1/bench_c2.json
