import time, torch, numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2511_04261_b200 as dp
ctx = dp.Context(0)
dev = torch.device('cuda:0')
for (M, N, C, b, n, ad) in [(576, 768, 3, 16, 1, False), (1080, 1920, 3, 16, 4, True)]:
    img = torch.zeros((1, M, N * C), dtype=torch.uint8, device=dev)
    out = torch.zeros_like(img)
    mask = torch.ones((1, M, N), dtype=torch.uint8, device=dev)
    d = dp._desc(M, N, C, 1)
    p = dp.make_privacy_params(0.5, 16, b, n)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(1, 1, C))
    G = dp.grid_dims(M, N, b).grid_count()
    cap = dp.adaptive_payload_capacity(M, N, b, n); st = (cap + 15)//16*16
    stats = torch.zeros((C, st), dtype=torch.uint8, device=dev)
    lens = torch.zeros(C, dtype=torch.int32, device=dev)
    def call():
        if ad: ctx.pixelize_adaptive_dev(d, img, mask, p, nz, stats, st, lens, out)
        else: ctx.pixelize_uniform_dev(d, img, p, nz, stats, out)
    for _ in range(20): call()
    ctx.synchronize()
    t0 = time.perf_counter(); K = 200
    for _ in range(K): call()
    t1 = time.perf_counter(); ctx.synchronize(); t2 = time.perf_counter()
    print(M, N, "issue us/call", (t1 - t0) / K * 1e6, "total us/call", (t2 - t0) / K * 1e6)
    # host-API call with pinned buffers
    h = torch.zeros((1, M, N, C), dtype=torch.uint8).pin_memory(); ho = torch.zeros_like(h).pin_memory()
    hm = torch.ones((1, M, N), dtype=torch.uint8).pin_memory()
    hs = torch.zeros((C, st), dtype=torch.uint8).pin_memory(); hl = torch.zeros(C, dtype=torch.int32).pin_memory()
    import ctypes as Ct
    def hcall():
        if ad: rc = dp._lib.dppx_pixelize_adaptive(ctx._h, Ct.byref(d), h.data_ptr(), hm.data_ptr(), Ct.byref(p), Ct.byref(nz), hs.data_ptr(), st, hl.data_ptr(), ho.data_ptr())
        else: rc = dp._lib.dppx_pixelize_uniform(ctx._h, Ct.byref(d), h.data_ptr(), Ct.byref(p), Ct.byref(nz), hs.data_ptr(), ho.data_ptr())
        assert rc == 0
    for _ in range(10): hcall()
    t0 = time.perf_counter(); K = 100
    for _ in range(K): hcall()
    t1 = time.perf_counter()
    print(M, N, "host-API us/call", (t1 - t0) / K * 1e6)
