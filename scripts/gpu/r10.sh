CFG=c1 bash scripts/gpu/ab_env.sh base NCSG_GA_CHUNKS=6 NCSG_GA_CHUNKS=12 NCSG_GA_CHUNKS=23
CFG=c5 bash scripts/gpu/ab_env.sh base NCSG_GA_CHUNKS=2
