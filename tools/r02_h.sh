# Sample stride experiment: key-only sample every R-th tile + main pass over all tiles.
O=gpurun_out/h; mkdir -p $O
for cfg in "--n 1000000 --d 64 --k 10 --fmt bf16" "--n 1000000 --d 64 --k 10 --fmt fp16"; do
  echo "== $cfg default"; timeout 300 python tools/prof_knn.py $cfg --reps 2 2>&1 | tail -1
  for R in 16 32 64; do
    echo "== $cfg keyonly R=$R"; TOD_SAMPLE_V1=0 TOD_SAMPLE_R=$R timeout 300 python tools/prof_knn.py $cfg --reps 2 2>&1 | tail -1
  done
done
echo "== c5s default"; timeout 300 python tools/prof_knn.py --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1
for R in 16 32; do echo "== c5s R=$R"; TOD_SAMPLE_R=$R timeout 300 python tools/prof_knn.py --n 500000 --d 512 --k 50 --fmt fp16 --reps 2 2>&1 | tail -1; done
echo "== c2 R=16"; TOD_SAMPLE_R=16 timeout 300 python tools/prof_knn.py --n 100000 --d 32 --k 20 --fmt fp16 --reps 3 2>&1 | tail -1
echo "== c2 default"; timeout 300 python tools/prof_knn.py --n 100000 --d 32 --k 20 --fmt fp16 --reps 3 2>&1 | tail -1
