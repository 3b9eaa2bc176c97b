# Look-ahead prefetch distance sweep (TDG_PF_TRACE / TDG_PF_FACE / TDG_PF_DOWN, blocks per SM)
for cfg in "4 4 4" "4 8 10" "2 8 10" "8 8 10" "4 4 10" "4 16 10" "4 8 5" "4 8 20" "4 12 14"; do
  set -- $cfg; export TDG_PF_TRACE=$1 TDG_PF_FACE=$2 TDG_PF_DOWN=$3
  echo "pf $cfg"; python tools/prof_residual.py --config 3 --n 32 --evals 10 | tail -1; python tools/prof_residual.py --config 4 --n 24 --evals 10 | tail -1
done
