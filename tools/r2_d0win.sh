# windowed d = 0 kernel: parity tests + C3 fp64 bench before/after (SLDG_SWEEP=r forces the register kernels)
O=gpurun_out/d0win; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "windowed_d0 or high_order_d0" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
B="--no-cpu-baseline --no-vlasov --no-compare-fp64"
timeout 300 python bench.py --config c3 --precision fp64 $B > $O/bench_c3_fp64.json 2> $O/bench_c3_fp64.err
timeout 300 python bench.py --config c3 --precision fp64 --k 5 $B > $O/bench_c3_fp64_k5.json 2> $O/bench_c3_fp64_k5.err
timeout 300 python bench.py --config c3 $B > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 python bench.py $B > $O/bench_c5.json 2> $O/bench_c5.err
