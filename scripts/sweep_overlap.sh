# sample || extract overlap knobs on the Papers pipeline (device-resident, no checksum)
CFG=papers timeout 600 python scripts/ab.py "S=6" "S=6,gather_evict_first=1" "S=6,gather_evict_first=2" "S=6,gather_evict_first=3" "S=6,cs=1" "S=6,cs=1,gather_evict_first=2" "S=6,cs=1,gather_evict_first=3" "S=5" "S=4" "S=6,l2_persist_mb=48" "S=6"
