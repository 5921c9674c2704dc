# Per-tile pipeline traces of the C2 main pass: session-start library vs the lean filter loop.
O=gpurun_out/s; mkdir -p $O
for lib in abl/base_libtod.so paper_2110_14007_b200/libtod.so; do
  echo "== $lib"
  TOD_MAIN_RING3=0 timeout 300 python tools/trace_main.py --lib $lib --n 100000 --d 32 --k 20 2>&1 | tail -16
done
