# Round-end style run: GPU tests, smoke, bench lines per config, ncu launch list + captures.
mkdir -p gpurun_out/prof
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/prof/pytest_gpu.txt 2>&1; tail -2 gpurun_out/prof/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/prof/smoke.txt 2>&1; tail -1 gpurun_out/prof/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/prof/bench_c2_line.json 2> gpurun_out/prof/bench_c2.err
timeout 900 python bench.py --config c3f16 --steps 5 --warmup 3 --no-cpu > gpurun_out/prof/bench_c3f16_line.json 2> /dev/null
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/prof/bench_c3_line.json 2> /dev/null
timeout 900 python bench.py --config c5s --steps 2 --warmup 3 --no-cpu > gpurun_out/prof/bench_c5s_line.json 2> /dev/null
timeout 600 python bench.py --config nwr --steps 10 --warmup 3 > gpurun_out/prof/bench_nwr_line.json 2> /dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/prof/bench_ref_line.json 2> /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c2_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc3 --launch-skip 1 -c 1 -o gpurun_out/prof/knn_tc3_c2 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rerank_groups -c 1 -o gpurun_out/prof/rerank_c2 python tools/prof_knn.py --n 100000 --d 32 --k 20 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc4 -c 1 -o gpurun_out/prof/knn_tc4_c3 python tools/prof_knn.py --n 1000000 --d 64 --k 10 --reps 1 > /dev/null 2>&1

timeout 300 python tools/dbg_modes.py > gpurun_out/prof/dbg_modes_c2.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/prof/bench_c2_torchrun1_line.json 2> gpurun_out/prof/torchrun.err
ls gpurun_out/prof
