# Per-group residual bounds in the re-rank; wave-balanced main-pass chunks; main-pass trace.
O=gpurun_out/d; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for f in "--n 100000 --d 32 --k 20 --fmt fp16 --reps 4" "--n 1000000 --d 64 --k 10 --fmt bf16 --reps 3" "--n 1000000 --d 64 --k 10 --fmt fp16 --reps 3" "--n 500000 --d 512 --k 50 --fmt fp16 --reps 2"; do
  echo "== $f"; timeout 300 python tools/prof_knn.py $f 2>&1 | tail -1; done
timeout 300 python tools/trace_main.py > $O/trace_c2.txt 2>&1; cat $O/trace_c2.txt
timeout 300 python tools/trace_main.py --n 1000000 --d 64 --k 10 > $O/trace_c3_1sm.txt 2>&1; cat $O/trace_c3_1sm.txt
timeout 300 python tools/dbg_modes.py > $O/dbg_modes_c2.txt 2>&1; cat $O/dbg_modes_c2.txt
timeout -s KILL 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "c3 or c2" > $O/pytest_full.txt 2>&1; tail -3 $O/pytest_full.txt
