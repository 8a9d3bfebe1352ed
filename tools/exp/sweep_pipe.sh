cd $GRAFT_REPO_ROOT
for lag in 60 80 100 140; do for ds in 20 40 80; do
  s=$((lag+ds))
  echo "== impl=2 LAG=$lag S=$s"
  BLOCKFFT_PIPE_IMPL=2 BLOCKFFT_PIPE_LAG=$lag BLOCKFFT_PIPE_S=$s timeout 60 python tools/time_variants.py --min 16 --max 16 --gib 2 --variants 5
done; done
