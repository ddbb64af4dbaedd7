# round 2: Amazon with 2048-element tiles (panel order) vs 1024, interleaved
set -x
mkdir -p gpurun_out
for t in 0 1 0 1; do
  echo "== BIG_TILES=$t" >> gpurun_out/r02w_tiles.log
  BLCO_B200_BIG_TILES=$t timeout 900 python scripts/panel_probe.py amazon "" >> gpurun_out/r02w_tiles.log 2>&1
done
