# Wave-balanced main-pass chunk count (default now): C2, C3, C4-shard-shape and d=128 A/B vs forced S.
O=gpurun_out/s8; mkdir -p $O
for rep in 1 2; do
  TOD_MAIN_S=1 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
  timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
done
TOD_MAIN_S=4 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 2>&1 | tail -1
timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 2>&1 | tail -1
timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "not c4 and not c5" > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $O/bench_c2_line.json 2> /dev/null; head -c 300 $O/bench_c2_line.json
