#!/bin/bash
# HEAD check: GPU tests, smoke, bench (N=1), 2-rank rehearsal, per-config timing, config-3 update split.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 2500 $OUT/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
tail -c 800 $OUT/bench_ref.json
timeout 600 python scripts/config_perf.py 2>&1 | tee $OUT/config_perf.txt
