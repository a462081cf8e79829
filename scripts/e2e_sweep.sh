mkdir -p gpurun_out
for ch in 262144 524288 1048576 2097152; do
  timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-chunk $ch 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($ch, d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['h2d_gbs'])"
done > gpurun_out/e2e_sweep.txt 2>&1
