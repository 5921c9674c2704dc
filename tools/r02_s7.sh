# Main-pass reference chunks S at C2 (782 query tiles on 148 SMs: the last wave is 42/148 full at S = 1).
for rep in 1 2; do
  for S in 1 2 3 5 7; do
    echo -n "S=$S "; TOD_MAIN_S=$S timeout 300 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
  done
done
