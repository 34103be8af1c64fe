O=gpurun_out/r2q; mkdir -p $O
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov"
bash tools/ab_run.sh . u1 _ab_u2 u2 c5 c5 c4 > $O/ab_unroll.txt 2>&1
(cd _ab_stamp && timeout 300 python bench.py --config c2 --steps 2 --warmup 3 $B --no-graph > $GRAFT_REPO_ROOT/$O/stamp_c2.json 2> $GRAFT_REPO_ROOT/$O/stamp_c2.err)
(cd _ab_stamp && timeout 300 python bench.py --config c3 --steps 1 --warmup 3 $B --no-graph > $GRAFT_REPO_ROOT/$O/stamp_c3.json 2> $GRAFT_REPO_ROOT/$O/stamp_c3.err)
(cd _ab_stamp && timeout 300 python bench.py --config c5 --steps 1 --warmup 1 $B --no-graph > $GRAFT_REPO_ROOT/$O/stamp_c5.json 2> $GRAFT_REPO_ROOT/$O/stamp_c5.err)
