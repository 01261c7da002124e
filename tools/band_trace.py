import sys, torch, ctypes as Ct
sys.path.insert(0, '/root/repo')
import paper_2511_04261_b200 as dp
ctx = dp.Context(0)
for (M, N, C, b, n) in [(2160, 3840, 3, 32, 8), (576, 768, 3, 16, 1)]:
    d = dp._desc(M, N, C, 1)
    p = dp.make_privacy_params(0.5, 16, b, n)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(1, 1, C))
    cap = dp.adaptive_payload_capacity(M, N, b, n); st = (cap + 15)//16*16
    h = torch.zeros((1, M, N, C), dtype=torch.uint8).pin_memory(); ho = torch.zeros_like(h).pin_memory()
    hm = torch.ones((1, M, N), dtype=torch.uint8).pin_memory()
    hs = torch.zeros((C, st), dtype=torch.uint8).pin_memory(); hl = torch.zeros(C, dtype=torch.int32).pin_memory()
    for it in range(3):
        print("call", M, N, it, file=sys.stderr, flush=True)
        if n > 1: rc = dp._lib.dppx_pixelize_adaptive(ctx._h, Ct.byref(d), h.data_ptr(), hm.data_ptr(), Ct.byref(p), Ct.byref(nz), hs.data_ptr(), st, hl.data_ptr(), ho.data_ptr())
        else: rc = dp._lib.dppx_pixelize_uniform(ctx._h, Ct.byref(d), h.data_ptr(), Ct.byref(p), Ct.byref(nz), hs.data_ptr(), ho.data_ptr())
        assert rc == 0
