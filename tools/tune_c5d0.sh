for dd in 2 3; do SLDG_TMA_D0DIV=$dd timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/t5_$dd.log 2>&1; done
timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/t4_new.log 2>&1
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/t2_new.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
