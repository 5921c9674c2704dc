# C2 re-rank with/without per-group residuals; C3 pair-kernel trace; C3 A/B of the eg default (bf16: on either way).
O=gpurun_out/y; mkdir -p $O
for rep in 1 2; do
  TOD_GROUP_EMAX=1 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
  timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
done
TOD_GROUP_EMAX=0 timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 2>&1 | tail -1
timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 2>&1 | tail -1
TOD_MAIN_PAIR=1 timeout 300 python tools/trace_main.py --n 1000000 --d 64 --k 10 --fmt bf16 2>&1 | tail -16
