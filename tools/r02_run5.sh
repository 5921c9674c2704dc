mkdir -p gpurun_out/r5
for v in "" "TOD_SAMPLE_R=16" "TOD_SAMPLE_V1=0" "TOD_SAMPLE_V1=0 TOD_SAMPLE_R=16"; do
  echo "== bf16 $v"; env $v python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 2>&1 | tail -1
  echo "== fp16 $v"; env $v python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt fp16 --reps 2 2>&1 | tail -1
done
for v in "" "TOD_SAMPLE_R=16"; do
  echo "== c2 $v"; env $v python tools/prof_knn.py --n 100000 --d 32 --k 20 --fmt fp16 --reps 3 2>&1 | tail -1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rerank_groups -c 1 -o gpurun_out/r5/rerank_c3bf16 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5/launches_c3_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
ls -la gpurun_out/r5
