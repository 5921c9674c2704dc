mkdir -p gpurun_out/r6
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r6/smi.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r6/bench_c3_line.json 2> gpurun_out/r6/bench_c3.err; tail -c 400 gpurun_out/r6/bench_c3_line.json
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/r6/bench_c2_line.json 2> gpurun_out/r6/bench_c2.err; tail -c 300 gpurun_out/r6/bench_c2_line.json
timeout 600 python bench.py --config c3f16 --steps 5 --warmup 3 --no-cpu > gpurun_out/r6/bench_c3f16_line.json 2> /dev/null
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r6/bench_c4_line.json 2> gpurun_out/r6/bench_c4.err; tail -c 300 gpurun_out/r6/bench_c4_line.json
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/r6/bench_c5_line.json 2> gpurun_out/r6/bench_c5.err; tail -c 300 gpurun_out/r6/bench_c5_line.json
timeout 600 python bench.py --config nwr --steps 10 --warmup 3 > gpurun_out/r6/bench_nwr_line.json 2> /dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r6/bench_ref_line.json 2> /dev/null
for mb in 48 24 16; do echo "== chunk $mb MB"; TOD_MAIN_CHUNK_MB=$mb python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 2 | tail -1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc4 -c 1 -o gpurun_out/r6/knn_tc4_c3bf16 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > /dev/null 2>&1
TOD_MAIN_CHUNK_MB=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc4 -c 1 -o gpurun_out/r6/knn_tc4_c3bf16_chunk16 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc -c 1 -o gpurun_out/r6/knn_tc_sample_c3bf16 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r6/launches_c2_bench.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
bash tools/r02_sanitize.sh > gpurun_out/r6/sanitize_summary.txt 2>&1; cat gpurun_out/r6/sanitize_summary.txt
timeout 1800 python bench.py --config c4 --loopback 8 --steps 1 --warmup 3 --no-cpu > gpurun_out/r6/bench_c4_loopback8_line.json 2> gpurun_out/r6/bench_c4_loopback8.err; tail -c 600 gpurun_out/r6/bench_c4_loopback8_line.json; tail -3 gpurun_out/r6/bench_c4_loopback8.err
