O=gpurun_out/r2r; mkdir -p $O
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov"
for v in _ab_stamp _ab_stamp0; do
  for c in c2 c3 c5; do
    st=2; [ $c = c5 ] && st=1
    (cd $v && timeout 300 python bench.py --config $c --steps $st --warmup 3 $B --no-graph > $GRAFT_REPO_ROOT/$O/${v}_$c.json 2> $GRAFT_REPO_ROOT/$O/${v}_$c.err)
  done
done
