# CTA-pair main pass with 160-column tiles x 3 accumulators (TOD_MAIN_NB=160).
O=gpurun_out/k; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ring3 or column or two_pass" > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for rep in 1 2; do
for nb in 160 256; do
 for cm in 0 1; do
  echo "== keyonly nb $nb colmode $cm"; TOD_SAMPLE_V1=0 TOD_MAIN_NB=$nb TOD_COLMODE=$cm timeout 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 2>&1 | tail -1
 done
done
done
echo "== default"; timeout 300 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 2>&1 | tail -1
TOD_SAMPLE_V1=0 TOD_MAIN_NB=160 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_knn_tc4 -c 1 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > $O/ncu_tc4_160.txt 2>&1; grep -E "duration|bytes|tensor" $O/ncu_tc4_160.txt
