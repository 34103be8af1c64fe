O=gpurun_out/r3c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vnodes.py -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for v in 1 0; do
  SLDG_VN_TMA=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-compare-fp64 --steps 2 > $O/bench_vn$v.json 2> $O/bench_vn$v.err
done
