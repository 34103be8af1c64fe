O=gpurun_out/vn; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vnodes.py -q -p no:cacheprovider > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-compare-fp64 > $O/bench_c5.json 2> $O/bench_c5.err
SLDG_VN_MULTI=0 timeout 300 python bench.py --no-cpu-baseline --no-compare-fp64 > $O/bench_c5_vn1.json 2> $O/bench_c5_vn1.err
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-compare-fp64 > $O/bench_c3.json 2> $O/bench_c3.err
SLDG_VN_MULTI=0 timeout 300 python bench.py --config c3 --no-cpu-baseline --no-compare-fp64 > $O/bench_c3_vn1.json 2> $O/bench_c3_vn1.err
