# Same-box A/B: round-start library (c54f482) vs the current one.
O=gpurun_out/o; mkdir -p $O
for rep in 1 2 3; do
  for lib in build/oldlib_libtod.so paper_2110_14007_b200/libtod.so; do
    timeout 300 python tools/ab_lib.py $lib --n 100000 --d 32 --k 20 --fmt fp16 2>&1 | tail -1
  done
done
for rep in 1 2; do
  for lib in build/oldlib_libtod.so paper_2110_14007_b200/libtod.so; do
    timeout 300 python tools/ab_lib.py $lib --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 2>&1 | tail -1
  done
done
