# Column candidates (release after the vote, columns re-read from TMEM): parity and timings.
O=gpurun_out/j; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for rep in 1 2; do
for cm in 1 0; do
  echo "== colmode $cm c3 bf16"; TOD_COLMODE=$cm timeout 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 2>&1 | tail -1
done
done
for cm in 1 0; do
  echo "== colmode $cm c5s"; TOD_COLMODE=$cm timeout 300 python tools/prof_knn.py --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
  echo "== colmode $cm c3 fp16"; TOD_COLMODE=$cm timeout 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt fp16 --reps 2 2>&1 | tail -1
done
echo "== c2"; timeout 300 python tools/prof_knn.py --n 100000 --d 32 --k 20 --fmt fp16 --reps 3 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_knn_tc4 -c 1 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > $O/ncu_tc4.txt 2>&1; grep -E "duration|bytes|tensor" $O/ncu_tc4.txt
