O=gpurun_out/vn3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vnodes.py -q -p no:cacheprovider > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-compare-fp64 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnode_sweep_multi -s 2 -c 1 -o $O/full_vn_multi_c5s python tools/diag_vnodes.py c5s > $O/ncu_multi.log 2>&1
