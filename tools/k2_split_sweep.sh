# K2 band-split A/B (DPPX_K2_SPLIT) over b = 32 / 64 grid sides, 120 x 1080p RGB adaptive
for bn in "32 1" "32 2" "32 4" "32 8" "64 1" "64 2" "64 4" "64 8" "64 16"; do
  for sp in 1 2 4; do echo "split=$sp $(DPPX_K2_SPLIT=$sp python tools/k2_case.py 1080 1920 120 $bn)"; done
done
for sp in 1 2 4; do echo "split=$sp 4K $(DPPX_K2_SPLIT=$sp python tools/k2_case.py)"; done
