O=gpurun_out/r2d; mkdir -p $O
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "bounded or bound_violation or timeline or graph or halo or transpose" > $O/pytest_new.log 2>&1; echo rc=$? >> $O/pytest_new.log
timeout 300 python bench.py $B > $O/bench_plain.json 2> $O/bench_plain.err
timeout 300 python bench.py $B --force-halo --timeline > $O/bench_halo.json 2> $O/bench_halo.err
timeout 300 python bench.py $B --force-halo --nccl-self --timeline > $O/bench_halo_nccl.json 2> $O/bench_halo_nccl.err
timeout 300 python bench.py --config c4 $B --force-halo --nccl-self --timeline > $O/bench_c4_halo_nccl.json 2> $O/bench_c4_halo_nccl.err
timeout 300 python bench.py --config c4 $B > $O/bench_c4_plain.json 2> $O/bench_c4_plain.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_strided -s 1 -c 1 -o $O/c5s_d1 python bench.py --dims 128,128,128,32 --sweeps 1 --steps 1 --warmup 1 $B --no-graph > $O/ncu_c5s_d1.log 2>&1
