set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2a_tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
timeout 900 python bench.py --gpus 2 --config products --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_g2.json 2> gpurun_out/r2a_g2.err
timeout 900 python bench.py --config mag --steps 20 --warmup 5 > gpurun_out/r2a_mag.json 2> gpurun_out/r2a_mag.err
tail -3 gpurun_out/*.err
