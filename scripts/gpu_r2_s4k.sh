# e2e: batch records' D2H on the extraction stream vs on a stream of their own.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host_seeds_e2e" > gpurun_out/s4k_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s4k_tests.txt
for rep in 1 2; do
  for v in 0 1; do
    timeout 900 python bench.py --no-cpu-baseline --no-per-call --option records_stream=$v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('records_stream=$v', round(d['value'],1), round(d['e2e']['value'],1), d['e2e']['device_ms'], d['clocks'])" >> gpurun_out/s4k_ab.txt
  done
done
