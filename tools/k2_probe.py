import sys, json, torch
sys.path.insert(0, '/root/repo')
import paper_2511_04261_b200 as dp
ctx = dp.Context(0)
dev = torch.device('cuda:0')
for F in (120, 600, 120):
    M, N, C, b, n = 1080, 1920, 3, 16, 4
    img = torch.empty((F, M, N*C), dtype=torch.uint8, device=dev); out = torch.empty_like(img)
    mask = torch.empty((F, M, N), dtype=torch.uint8, device=dev)
    d = dp._desc(M, N, C, F); ctx.synth_frames_dev(d, 101, 0, img, mask)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    p = dp.make_privacy_params(0.5, 16, b, n)
    cap = dp.adaptive_payload_capacity(M, N, b, n); st = (cap + 15)//16*16
    stats = torch.zeros((F*C, st), dtype=torch.uint8, device=dev); lens = torch.zeros(F*C, dtype=torch.int32, device=dev)
    ctx.pixelize_adaptive_dev(d, img, mask, p, nz, stats, st, lens, out); ctx.synchronize()
    for rep in range(2):
        ctx.reset_stats(); ctx.set_timing(True)
        for _ in range(3): ctx.reassemble_dev(d, stats, st, lens, b, n, out)
        ctx.synchronize(); s = ctx.stats(); ctx.set_timing(False)
        k2 = s['device_ms']['expand'] / s['launches']['expand']; k0 = s['device_ms']['classify'] / max(1, s['launches']['classify'])
        alg = F*M*N*C + int(lens.sum().item())
        print(F, rep, 'k2 ms', round(k2, 4), 'frac', round(alg/(k2/1e3)/1e9/6543.1, 3), 'k0 ms', round(k0, 4))
    del img, out, mask, stats
