O=gpurun_out/hik; mkdir -p $O
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov --no-graph"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_d0 -s 3 -c 1 -o $O/full_d0_k5 python bench.py --steps 1 --warmup 3 $B --config c3 --k 5 > $O/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_strided -s 3 -c 1 -o $O/full_st_k5 python bench.py --steps 1 --warmup 3 $B --config c3 --k 5 > $O/ncu2.log 2>&1
