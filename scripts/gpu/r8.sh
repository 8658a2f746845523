bash scripts/gpu/allcfg.sh NCSG_X=1
CFGS="c1 c3" bash scripts/gpu/allcfg.sh NCSG_EAGER=1
