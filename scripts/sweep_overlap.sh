# gather engine choices inside the Papers / Friendster pipeline (device-resident, no checksum)
for c in papers friendster; do
CFG=$c timeout 600 python scripts/ab.py "S=8" "S=8,gather_impl=3" "S=8,mode=extract" "S=8,mode=extract,gather_impl=3"
done
