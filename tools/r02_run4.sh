mkdir -p gpurun_out/r4
python tools/prof_knn.py --n 100000 --d 32 --k 20 --fmt fp16 --reps 3 2>&1 | tail -1
python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 3 2>&1 | tail -1
python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt fp16 --reps 2 2>&1 | tail -1
python tools/prof_knn.py --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
timeout -s KILL 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_certificate.py -q -p no:cacheprovider -x > gpurun_out/r4/pytest.txt 2>&1; tail -3 gpurun_out/r4/pytest.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r4/bench_c3.json 2> gpurun_out/r4/bench_c3.err; tail -c 1200 gpurun_out/r4/bench_c3.json
timeout 1200 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu > gpurun_out/r4/bench_c4.json 2> gpurun_out/r4/bench_c4.err; tail -c 900 gpurun_out/r4/bench_c4.json
bash tools/r02_sanitize.sh
