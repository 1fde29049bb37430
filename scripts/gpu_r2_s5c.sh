# per_call variance: the reference-shaped per-call SET loop alone, three times.
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 600 tools/set_loop --generate 111059956:128:16:7 4444000 200 2>&1 | grep per_call >> gpurun_out/s5c_percall.txt
done
