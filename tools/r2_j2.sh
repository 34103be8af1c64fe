# A/B of the two-slots-per-iteration k >= 5 d = 0 consumer: default build, then -DSLDG_D0_J2=1 built on the box
O=gpurun_out/j2; mkdir -p $O
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov"
ab() {  # ab <tag>
  for k in 5 6; do
    timeout 300 python bench.py --config c3 --k $k $B > $O/$1_mixed_k$k.json 2>/dev/null
    timeout 300 python bench.py --config c3 --k $k --precision fp64 $B > $O/$1_fp64_k$k.json 2>/dev/null
  done
}
ab base
SLDG_NVCC_EXTRA="-DSLDG_D0_J2=1" python -m paper_1603_07008_b200._build --force > $O/build_j2.log 2>&1
ab j2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "high_order_d0 or windowed_d0 or single_sweeps" > $O/pytest_j2.log 2>&1; echo rc=$? >> $O/pytest_j2.log
ab j2b
