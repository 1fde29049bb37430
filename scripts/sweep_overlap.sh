# 64-byte L2 fetch hint on table reads (gather_pf64) for 400-byte (products) and 512-byte (Papers) rows
CFG=products K=196 timeout 600 python scripts/ab.py "S=8" "S=8,gather_pf64=1" "S=8,mode=extract" "S=8,mode=extract,gather_pf64=1" "S=8,cs=1" "S=8,cs=1,gather_pf64=1"
CFG=papers timeout 600 python scripts/ab.py "S=8" "S=8,gather_pf64=1" "S=8,mode=extract" "S=8,mode=extract,gather_pf64=1"
