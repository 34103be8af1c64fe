# Bench lines for profiles/round1 (run under gpurun): every config (mixed; fp64 where it fits),
# the eps = 0.5 stress fields for C2 and C5, the reference arm, smoke().
O=gpurun_out/fb
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for c in c5 c4 c3 c2; do python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in c4 c3 c2; do python bench.py --config $c --precision fp64 > $O/bench_${c}_fp64.json 2> $O/bench_${c}_fp64.err; done
for c in c5 c2; do python bench.py --config $c --eps 0.5 > $O/bench_${c}_eps05.json 2> $O/bench_${c}_eps05.err; done
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for f in $O/*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['value'],3), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'))"; done
cat $O/smoke.log | tail -2
