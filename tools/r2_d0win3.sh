O=gpurun_out/d0win3; mkdir -p $O
B="--no-cpu-baseline --no-vlasov --no-compare-fp64"
for k in 2 3 4 5 6; do
  SLDG_D0_WIN=1 timeout 300 python bench.py --config c3 --k $k $B > $O/win_c3_mixed_k$k.json 2> $O/win_c3_mixed_k$k.err
  timeout 300 python bench.py --config c3 --k $k $B > $O/base_c3_mixed_k$k.json 2> $O/base_c3_mixed_k$k.err
done
for k in 5 6; do
  SLDG_TMA_F64HI=1 timeout 300 python bench.py --config c3 --precision fp64 --k $k $B > $O/f64hi_c3_fp64_k$k.json 2> $O/f64hi_c3_fp64_k$k.err
  timeout 300 python bench.py --config c3 --precision fp64 --k $k $B > $O/base_c3_fp64_k$k.json 2> $O/base_c3_fp64_k$k.err
done
