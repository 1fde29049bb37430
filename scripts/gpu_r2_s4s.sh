# Products / Papers: gather CTAs per SM per launch.
mkdir -p gpurun_out
for rep in 1 2; do
  CFG=products K=196 timeout 900 python scripts/ab.py "S=8" "S=8,gather_ctas_per_sm=2" "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4s_ab.txt
  K=300 timeout 900 python scripts/ab.py "S=8" "S=8,gather_ctas_per_sm=2" 2>&1 | grep us/batch >> gpurun_out/s4s_ab.txt
done
