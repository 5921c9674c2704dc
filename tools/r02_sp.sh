# Key-only sample pass on the K-pipelined CTA pair (dpad > 64): parity + A/B (TOD_SAMPLE_PAIR=0/1).
O=gpurun_out/sp; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "kpipelined or high_dimensional or column" > $O/pytest_sp.txt 2>&1; tail -3 $O/pytest_sp.txt
for rep in 1 2; do
  TOD_SAMPLE_PAIR=0 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
  TOD_SAMPLE_PAIR=1 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
done
TOD_SAMPLE_PAIR=0 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
TOD_SAMPLE_PAIR=1 timeout 600 python tools/ab_lib.py paper_2110_14007_b200/libtod.so --n 200000 --d 128 --k 10 --fmt fp16 --reps 3 2>&1 | tail -1
