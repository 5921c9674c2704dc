# Re-rank pre-bound, unrolled (compile-time dpad, 4 partial sums): A/B at C2, C3 bf16/fp16, d=128.
O=gpurun_out/pb2; mkdir -p $O
for rep in 1 2; do
  TOD_RR_PREBOUND=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
  timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
done
for f in bf16 fp16; do
  TOD_RR_PREBOUND=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 64 --k 10 --fmt $f --reps 2 2>&1 | tail -1
  timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 64 --k 10 --fmt $f --reps 2 2>&1 | tail -1
done
TOD_RR_PREBOUND=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
