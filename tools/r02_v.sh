# Re-rank profiles (C2 fp16, C3 bf16) with source attribution; C2 bench line with knn_tc3 default.
O=gpurun_out/v; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rerank_groups -c 1 -o $O/rerank_c2 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rerank_groups -c 1 -o $O/rerank_c3 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > /dev/null 2>&1
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $O/bench_c2_line.json 2> $O/bench_c2.err; head -c 400 $O/bench_c2_line.json
ls $O
