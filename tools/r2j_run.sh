O=gpurun_out/r2j; mkdir -p $O
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov"
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x -p no:cacheprovider > $O/pytest_fused.log 2>&1; echo rc=$? >> $O/pytest_fused.log
for c in c5 c4; do
  timeout 300 python bench.py --config $c $B > $O/${c}_plain.json 2> $O/${c}_plain.err
  timeout 300 python bench.py --config $c $B --fuse-x > $O/${c}_fused.json 2> $O/${c}_fused.err
done
