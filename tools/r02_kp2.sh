# C5-shape A/B with candidate statistics: single-SM vs CTA-pair K-pipelined main pass.
for rep in 1; do
  TOD_MAIN_PAIR=0 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
  TOD_MAIN_PAIR=1 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
  TOD_COLMODE=0 TOD_MAIN_PAIR=0 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
  TOD_COLMODE=0 TOD_MAIN_PAIR=1 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
done
