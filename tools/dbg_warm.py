import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1802_08021_b200 import sparcml as S
N, k = 1 << 20, 10_000
for ef in (False, True):
    ws = S.TopkWorkspace(N, k)
    rng = np.random.default_rng(21)
    for it, scale in enumerate([1.0, 1.0, 1e-3, 1.0, 1.0, 1e3, 1.0]):
        x = torch.from_numpy((rng.standard_normal(N) * scale).astype(np.float32)).cuda()
        if ef:
            g = torch.from_numpy((rng.standard_normal(N) * scale).astype(np.float32)).cuda()
            S.ef_topk(x, g, 0.5, k, ws=ws)
        else:
            res = torch.empty(N, device="cuda")
            S.topk_sparsify(x, k, residual=res, ws=ws)
        torch.cuda.synchronize()
        w = ws.buf[221632:221656].cpu().numpy()
        print(ef, it, scale, ws.status(), hex(int(w[:4].view(np.uint32)[0])), int(w[4:8].view(np.uint32)[0]), int(w[8:16].view(np.uint64)[0]), int(w[16:24].view(np.uint64)[0]), "bytes", ws.bytes)
