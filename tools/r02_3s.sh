# Three-stage selection at d <= 32 on the single-SM kernel: parity + A/B (TOD_SAMPLE3=0/1) at C2.
O=gpurun_out/3s; mkdir -p $O
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $O/pytest_parity.txt 2>&1; tail -3 $O/pytest_parity.txt
for rep in 1 2 3; do
  TOD_SAMPLE3=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
  TOD_SAMPLE3=1 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
done
TOD_SAMPLE3=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 32 --k 10 --fmt fp16 --reps 2 2>&1 | tail -1
TOD_SAMPLE3=1 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 32 --k 10 --fmt fp16 --reps 2 2>&1 | tail -1
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $O/bench_c2_line.json 2> $O/bench_c2.err; head -c 300 $O/bench_c2_line.json
