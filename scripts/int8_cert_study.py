# CPU numerics experiment: certified int8 (per-128-row-tile scale) shortlist sizes at 1M x 768
import torch, numpy as np, time, sys
torch.manual_seed(0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
D, NQ, K, TILE = 768, 256, 8, 128
g = torch.Generator().manual_seed(1)
X = torch.randn(N, D, generator=g)
X = X / X.double().norm(dim=1, keepdim=True).float()
nd = N // 20
src = torch.randint(0, N // 2, (nd,), generator=g)
dst = N // 2 + torch.randperm(N - N // 2, generator=g)[:nd]
X[dst] = X[src]
q = torch.randn(NQ, D, generator=g)
h = NQ // 2
s = torch.randint(0, N, (h,), generator=g)
u = torch.randn(h, D, generator=g); u = u / u.norm(dim=1, keepdim=True)
sig = torch.rand(h, 1, generator=g) * 1.25
q[:h] = X[s] + sig * u
q = q / q.double().norm(dim=1, keepdim=True).float()

def quant_tiles(X, tile):
    n = X.shape[0]
    pad = (-n) % tile
    Xp = torch.cat([X, torch.zeros(pad, X.shape[1])]) if pad else X
    Xt = Xp.view(-1, tile, X.shape[1])
    st = Xt.abs().amax(dim=(1, 2)) / 127.0
    Xq = torch.round(Xt / st[:, None, None]).clamp(-127, 127)
    deq = Xq * st[:, None, None]
    err = (Xt.double() - deq.double()).norm(dim=2)  # per row ||dx||
    return Xq.view(-1, X.shape[1])[:n], st.repeat_interleave(tile)[:n], err.view(-1)[:n]

t0 = time.time()
Xq, sx, ex = quant_tiles(X, TILE)
qs = q.abs().amax(dim=1) / 127.0
qq = torch.round(q / qs[:, None]).clamp(-127, 127)
eq = (q.double() - (qq * qs[:, None]).double()).norm(dim=1)
qhat_norm = (qq.double() * qs[:, None].double()).norm(dim=1)
xnorm = X.double().norm(dim=1)
print("quant done", time.time() - t0, "max ||dx||", ex.max().item(), "median", ex.median().item(), "max ||dq||", eq.max().item())
# int dots exact in fp32 (|partial| < 2^24)
dots = qq @ Xq.T                      # [NQ][N]
approx = dots.double() * qs[:, None].double() * sx[None, :].double()
exact = (q @ X.T).double()            # fine for counting
Tk = exact.topk(K, dim=1).values[:, -1]
eps_glob = eq * xnorm.max() + qhat_norm * ex.max() + 1e-6
err_actual = (approx - exact).abs().max().item()
need = (approx >= (Tk - eps_glob)[:, None]).sum(dim=1)
print("actual max |approx-exact|", err_actual, "eps median", eps_glob.median().item())
print("int8 needed shortlist: median", need.median().item(), "p90", need.float().quantile(0.9).item(), "p99", need.float().quantile(0.99).item(), "max", need.max().item())
# bf16 comparison
Xb = X.bfloat16().float(); qb = q.bfloat16().float()
dxb = (X.double() - Xb.double()).norm(dim=1).max(); dqb = (q.double() - qb.double()).norm(dim=1)
apb = (qb @ Xb.T).double()
epsb = dxb + dqb * (1 + dxb) + 2**-13 * 2.1
needb = (apb >= (Tk - epsb)[:, None]).sum(dim=1)
print("bf16 eps", epsb.median().item(), "needed: median", needb.median().item(), "p99", needb.float().quantile(0.99).item(), "max", needb.max().item())
# fresh vs perturbed split
print("Tk median", Tk.median().item())
