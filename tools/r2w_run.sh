O=gpurun_out/r2w; mkdir -p $O
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov"
for v in _ab_stamp _ab_stampw; do
  for c in c2 c3; do
    (cd $v && timeout 300 python bench.py --config $c --steps 2 --warmup 3 $B --no-graph > $GRAFT_REPO_ROOT/$O/${v}_$c.json 2> $GRAFT_REPO_ROOT/$O/${v}_$c.err)
  done
done
