#!/bin/bash
# Every bench.py line of the round into gpurun_out/bench_r2/ (run on the GPU box).
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/bench_r2
mkdir -p $out
python bench.py --steps 10 --warmup 3 > $out/bench_c2.json 2> $out/bench_c2.err
python bench.py --config c1 --steps 10 --warmup 3 > $out/bench_c1.json 2> $out/bench_c1.err
python bench.py --config c5 --steps 10 --warmup 3 > $out/bench_c5.json 2> $out/bench_c5.err
python bench.py --config c3 --steps 5 --warmup 3 > $out/bench_c3.json 2> $out/bench_c3.err
python bench.py --dtype c64 --steps 10 --warmup 3 --no-sparse > $out/bench_c2_c64.json 2> $out/bench_c2_c64.err
python bench.py --config c4 --warmup 3 > $out/bench_c4.json 2> $out/bench_c4.err
python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref_c2.json 2> $out/bench_ref_c2.err
for f in $out/*.json; do echo "== $f"; tail -c 400 $f; echo; done
