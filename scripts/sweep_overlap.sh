# sample || extract overlap knobs on the Papers pipeline (device-resident, no checksum)
CFG=papers timeout 600 python scripts/ab.py "S=6" "S=6,gather_evict_first=0" "S=8,gather_evict_first=0" "S=6,gather_evict_first=0,hash_keep=0" "S=6,cs=1" "S=6,cs=1,gather_evict_first=0" "S=6,mode=extract,gather_evict_first=0" "S=6,mode=extract,cs=1,gather_evict_first=0" "S=6,mode=extract,cs=1"
CFG=friendster timeout 600 python scripts/ab.py "S=6" "S=6,gather_evict_first=0" "S=6,cs=1" "S=6,cs=1,gather_evict_first=0"
