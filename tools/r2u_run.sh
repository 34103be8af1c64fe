O=gpurun_out/r2u; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fused.py -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
bash tools/env_sweep.sh SLDG_WALK "1 0 1 0" c5 c4 c3 > $O/walk.txt 2>&1
