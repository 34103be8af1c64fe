O=gpurun_out/r2n; mkdir -p $O
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov"
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x -p no:cacheprovider > $O/pytest_fused.log 2>&1; echo rc=$? >> $O/pytest_fused.log
for st in 2 3; do
  SLDG_FUSED_STAGES=$st timeout 300 python bench.py --config c5 $B --fuse-x > $O/c5_fused_s$st.json 2> $O/c5_fused_s$st.err
done
SLDG_FUSED_STAGES=2 SLDG_FUSED_TSUB=7 timeout 300 python bench.py --config c5 $B --fuse-x > $O/c5_fused_s2r8.json 2> $O/c5_fused_s2r8.err
timeout 300 python bench.py --config c4 $B --fuse-x > $O/c4_fused.json 2> $O/c4_fused.err
timeout 300 python bench.py --config c5 $B > $O/c5_plain.json 2> $O/c5_plain.err
