# A/B: segsum warp slices per SM (FK_SEGSUM_WPS), configs 3, 2, 4.
mkdir -p gpurun_out
for r in 1 2; do
  for w in 32 24 16; do echo "wps=$w:"; FK_SEGSUM_WPS=$w SHAPE=4,0,1 python scripts/update_small.py; done
done > gpurun_out/ab_seg2.txt 2>&1
