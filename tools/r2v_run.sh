O=gpurun_out/r2v; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_vlasov.py -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
bash tools/ab_run.sh _ab_fz0 widen . promo c5 c5 c4 > $O/ab.txt 2>&1
