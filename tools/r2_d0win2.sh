O=gpurun_out/d0win2; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
B="--no-cpu-baseline --no-vlasov --no-compare-fp64"
for k in 2 3 4 5 6; do
  timeout 300 python bench.py --config c3 --precision fp64 --k $k $B > $O/bench_c3_fp64_k$k.json 2> $O/bench_c3_fp64_k$k.err
  timeout 300 python bench.py --config c3 --k $k $B > $O/bench_c3_mixed_k$k.json 2> $O/bench_c3_mixed_k$k.err
done
timeout 300 python bench.py --config c3 --precision fp64 $B --dims 4100,4096 > $O/bench_c3_fp64_4100.json 2> $O/bench_c3_fp64_4100.err
