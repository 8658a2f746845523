CFG=c2 bash scripts/gpu/ab_lib.sh base r8 c4 c1
CFG=c3 bash scripts/gpu/ab_lib.sh base r8 c4 c1
