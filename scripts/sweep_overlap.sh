# sample || extract overlap knobs on the Papers pipeline (device-resident, no checksum)
CFG=papers timeout 600 python scripts/ab.py "S=6" "S=6,cs=1" "S=8" "S=6,mode=sample" "S=6"
