# Out-of-core tier: prefetch-size hints on the zero-copy row reads (PCIe request size).
mkdir -p gpurun_out
for pf in 0 2 1; do
  timeout 1200 python bench.py --config papers_host_bm --steps 20 --warmup 5 --no-cpu-baseline --no-per-call --option host_tier_pf=$pf 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pf=$pf', round(d['value'],1), d['host_tier'])" >> gpurun_out/s5b_ab.txt
done
