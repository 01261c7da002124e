# A/B of two builds (_ab/old, _ab/new) over the b sweeps (60 frames)
for v in old new; do echo "== $v"; DPPX_LIB=_ab/$v/libdppx_gpu.so python tools/b_sweep.py 60 uniform 2>&1 | tail -22; DPPX_LIB=_ab/$v/libdppx_gpu.so python tools/b_sweep.py 60 2>&1 | tail -31; done
