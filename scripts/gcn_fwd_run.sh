# K3 gather-warp count sweep (libraries from scripts/gcn_fwd_roles.sh)
for rep in 1 2; do
  for g in ${G:-12 16 20 24 26}; do DGNN_LIB_PATH=$PWD/scripts/probe_libs/libgtc_$g.so timeout 120 python scripts/gcn_fwd_probe.py; done
done
