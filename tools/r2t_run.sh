O=gpurun_out/r2t; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -m gpu -q -x -p no:cacheprovider -k "graph or halo or transpose or bounded or pair or c2 or single_sweeps or randomized_shapes" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
bash tools/env_sweep.sh SLDG_PDL "1 0 1 0" c2 c3 c4 c5 > $O/pdl.txt 2>&1
