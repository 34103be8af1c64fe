# peer-mapped halos on one GPU: tests + C5 bench lines (plain, copy halo, peer halo)
O=gpurun_out/peer; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_peer_host.py -q -p no:cacheprovider -x > $O/pytest_peer.log 2>&1; echo rc=$? >> $O/pytest_peer.log
B="--no-cpu-baseline --no-vlasov --no-compare-fp64"
timeout 300 python bench.py $B > $O/bench_plain.json 2> $O/bench_plain.err
timeout 300 python bench.py $B --force-halo > $O/bench_halo_copy.json 2> $O/bench_halo_copy.err
timeout 300 python bench.py $B --peer-halo > $O/bench_halo_peer.json 2> $O/bench_halo_peer.err
timeout 300 python bench.py $B --peer-halo --timeline > $O/bench_halo_peer_tl.json 2> $O/bench_halo_peer_tl.err
timeout 300 python bench.py $B > $O/bench_plain2.json 2> $O/bench_plain2.err
