# Staggered sweep start (TileSeq rotation) A/B, vote flag, TMEM read throughput.
O=gpurun_out/c; mkdir -p $O
timeout 120 ./build/tmem_bench > $O/tmem_bench.txt 2>&1; cat $O/tmem_bench.txt
for st in 1 0; do
 for f in "--n 100000 --d 32 --k 20 --fmt fp16 --reps 4" "--n 1000000 --d 64 --k 10 --fmt bf16 --reps 3" "--n 500000 --d 512 --k 50 --fmt fp16 --reps 2"; do
  echo "== stagger $st $f"; TOD_STAGGER=$st timeout 300 python tools/prof_knn.py $f 2>&1 | tail -1; done
done
echo "== c2 vote 1"; TOD_VOTE=1 timeout 300 python tools/prof_knn.py --n 100000 --d 32 --k 20 --fmt fp16 --reps 4 2>&1 | tail -1
timeout 300 python tools/dbg_modes.py > $O/dbg_modes_c2.txt 2>&1; cat $O/dbg_modes_c2.txt
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
