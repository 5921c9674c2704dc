./tools/tmem_bench
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc -c 1 -o gpurun_out/knn_tc_c2 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 > gpurun_out/ncu_c2.log 2>&1; tail -2 gpurun_out/ncu_c2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc -c 1 -o gpurun_out/knn_tc_c3 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 1 > gpurun_out/ncu_c3.log 2>&1; tail -2 gpurun_out/ncu_c3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/b_ncu.log 2>&1
