"""Fraction of kmeans points the kmeans_tg screen defers (several candidates
within 2E), for the first centroids (first 16 points) and for the centroids
of later Lloyd passes: 16M x 32 U(0,1), k = 16, the bench's data shape.
`old`: the round-2 two-plane bound (E = 2^-12 |f| cmax + 2^-17 cmax^2);
`new`: three centroid planes (E = 2^-14 |f| cmax + 2^-21 cmax^2)."""
import torch
torch.manual_seed(0)
npts, nf, k = 1 << 24, 32, 16
f = torch.rand(nf, npts, device="cuda")
c = f[:, :k].t().contiguous()
fd = f.double()
n2 = (fd * fd).sum(0)
for it in range(11):
    cd = c.double()
    cn = (cd * cd).sum(1)
    cmax = cn.max().sqrt().item() * 1.001
    eA = 2.44140625e-4 * 1.01 * cmax
    eB = 7.62939453125e-06 * cmax * cmax
    eA2 = 6.103515625e-05 * 1.01 * cmax
    eB2 = 4.76837158203125e-07 * cmax * cmax
    tv = cn[None, :] - 2.0 * (fd.t() @ cd.t())          # [npts, k]
    E = eA * n2.sqrt() + eB + 9.2e-13 * n2
    E2 = eA2 * n2.sqrt() + eB2 + 9.2e-13 * n2
    mn, best = tv.min(1)
    cand = (tv <= (mn + 2 * E)[:, None]).sum(1)
    srt = tv.sort(1).values
    gap = srt[:, 1] - srt[:, 0]
    cand2 = (tv <= (mn + 2 * E2)[:, None]).sum(1)
    print(f"pass {it}: new bound deferred {(cand2 > 1).float().mean().item():.5f} ({int((cand2 > 1).sum())} pts); "
          f"old deferred {(cand > 1).float().mean().item():.5f} ({int((cand > 1).sum())} pts), "
          f"mean cand {cand.float().mean().item():.4f}, 2E median {2 * E.median().item():.2e}, "
          f"gap p1 {gap.kthvalue(npts // 100).values.item():.2e}, "
          f"defer at E/8 {((tv <= (mn + E / 4)[:, None]).sum(1) > 1).float().mean().item():.5f}")
    # Lloyd update
    cnt = torch.bincount(best, minlength=k).double()
    s = torch.zeros(k, nf, dtype=torch.float64, device="cuda").index_add_(0, best, fd.t())
    c = (s / cnt[:, None].clamp(min=1)).float()
