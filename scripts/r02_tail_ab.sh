python scripts/norm_tail_perf.py 2>&1 | tail -2
for v in fused split; do echo "== FK_TAIL=$v"; FK_TAIL=$v python scripts/norm_tail_perf.py 2>&1 | tail -2; done
python scripts/config_perf.py 2>&1 | tail -4
