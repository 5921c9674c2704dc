# Round-2 final evidence at HEAD (outputs kept small: ncu reports summarised to text on the box).
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 -rf > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_c3_line.json 2> $O/bench_c3.err; head -c 200 $O/bench_c3_line.json; echo
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $O/bench_c2_line.json 2> $O/bench_c2.err; head -c 200 $O/bench_c2_line.json; echo
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 > $O/bench_c4_line.json 2> $O/bench_c4.err; head -c 200 $O/bench_c4_line.json; echo
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 > $O/bench_c5_line.json 2> $O/bench_c5.err; head -c 200 $O/bench_c5_line.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref_line.json 2> /dev/null; head -c 200 $O/bench_ref_line.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_bench.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
cap() {  # name, kernel regex, skip, args...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre --launch-skip $skip -c 1 -o /tmp/$name python tools/prof_knn.py "$@" > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep > $O/${name}_full.txt 2>&1
  python tools/stalls.py /tmp/$name.ncu-rep > $O/${name}_stalls.txt 2>&1
  rm -f /tmp/$name.ncu-rep
}
cap knn_tc4_c3bf16 k_knn_tc4 1 --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1
cap knn_tc3_c2 k_knn_tc3 1 --n 100000 --d 32 --k 20 --reps 1
cap knn_tc4_d512 k_knn_tc4 0 --n 200000 --d 512 --k 50 --reps 1
cap rerank_c3 k_rerank_groups 0 --n 1000000 --d 64 --k 10 --fmt bf16 --reps 1
du -sh $O; ls $O
