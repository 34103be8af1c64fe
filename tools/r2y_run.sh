O=gpurun_out/r2y; mkdir -p $O
timeout 600 python tools/order_sweep.py --reps 5 --out $O/order_spl3.md > $O/spl3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "high_order or randomized or single_sweeps or c3" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
