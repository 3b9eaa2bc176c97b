# k_mortar register-cap sweep (resident one-warp blocks per SM), config-3 residual split
for cfg in "16 20" "20 24" "24 24" "24 32" "32 32"; do
  set -- $cfg
  TDG_NVCC_EXTRA="-DTDG_MORTAR_BLOCKS_FLUX=$1 -DTDG_MORTAR_BLOCKS_LIFT=$2" python -m paper_1806_11456_b200.build --force 2>&1 | grep "k_mortar" | sed 's/.*function//'
  echo "flux blocks $1 lift blocks $2"
  python tools/prof_residual.py --config 3 --n 32 --evals 5 2>&1 | tail -1
done
