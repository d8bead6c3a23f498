"""Round-2 design aid (not product code, not a test): numpy simulation of the
fp32 error of the one-pass tensor-core affine MLS (F = sum_m c_m (w phi_m) Q)
against the current two-pass form (F = [w (c0 + c1 dx + c2 dy)] Q), with the
same tf32 hi/lo splits and 512-control fp32 runs into fp64 totals, on a
config-3-shaped frame (GMM 100k x 32, 3840x2160, sampled pixels).  Only the
ratio of the two errors is meaningful: the simulated input rounding is
coarser than the kernel's.  DESIGN.md "Next" item 0.
"""
import numpy as np
rng = np.random.default_rng(3)
N, d, K = 100_000, 32, 8
cent = rng.normal(0, 4, (K, d)); sc = rng.uniform(0.5, 1.5, K); lab = rng.integers(0, K, N)
X = cent[lab] + sc[lab, None] * rng.normal(size=(N, d))
Xn = (X - X.mean(0)) / X.std(0)
C = np.cov(Xn.T); ev, V = np.linalg.eigh(C); P = Xn @ V[:, ::-1][:, :2]
Q = X.copy()
lo, hi = P.min(0), P.max(0); pad = 0.05 * (hi - lo); lo -= pad; hi += pad
W, H = 3840, 2160
npx = 600
ii = np.concatenate([rng.integers(0, W, npx - 8), [0, W-1, 0, W-1, W//2, 0, W-1, W//2]])
jj = np.concatenate([rng.integers(0, H, npx - 8), [0, 0, H-1, H-1, 0, H//2, H//2, H-1]])
vx = lo[0] + (ii + .5) * (hi[0]-lo[0]) / W; vy = hi[1] - (jj + .5) * (hi[1]-lo[1]) / H
pm = P.mean(0); qm = Q.mean(0)
Pc = P - pm; Qc = Q - qm; vx = vx - pm[0]; vy = vy - pm[1]
f32 = np.float32
def tf32_split(a):
    a = a.astype(f32); b = a.view(np.uint32) & np.uint32(0xFFFFE000); h = b.view(f32); return h, (a - h).astype(f32)
Qh, Ql = tf32_split(Qc)
def runsum(T, run=512):  # fp32 sums over runs, fp64 totals; T: (N, ...) fp32 terms
    out = 0.0
    for s in range(0, N, run):
        out = out + np.sum(T[s:s+run], axis=0, dtype=f32).astype(np.float64)
    return out
errs_two, errs_one = [], []
ref_all, two_all, one_all = [], [], []
for p in range(npx):
    dx = Pc[:, 0] - vx[p]; dy = Pc[:, 1] - vy[p]
    d2 = dx*dx + dy*dy; w = d2 ** -1.5
    A = np.array([[w.sum(), (w*dx).sum(), (w*dy).sum()], [0, (w*dx*dx).sum(), (w*dx*dy).sum()], [0, 0, (w*dy*dy).sum()]])
    A[1,0], A[2,0], A[2,1] = A[0,1], A[0,2], A[1,2]
    S = A[1:,1:] - np.outer(A[1:,0], A[0,1:]) / A[0,0]; r = 1e-12 * np.trace(S)
    Ar = A + np.diag([0, r, r]); c = np.linalg.solve(Ar, np.array([1., 0, 0]))
    ref = (w * (c[0] + c[1]*dx + c[2]*dy)) @ Qc
    # fp32 simulation (moments in fp64 here: both schemes share pass-1 accuracy)
    dx32 = (Pc[:, 0].astype(f32) - f32(vx[p])); dy32 = (Pc[:, 1].astype(f32) - f32(vy[p]))
    w32 = ((dx32*dx32 + dy32*dy32) ** f32(-1.5)).astype(f32)
    c32 = c.astype(f32)
    G = w32 * (c32[0] + c32[1]*dx32 + c32[2]*dy32)
    Gh, Gl = tf32_split(G)
    two = runsum(Gh[:, None]*Qh + Gh[:, None]*Ql + Gl[:, None]*Qh)
    T = 0.0
    for m, phi in enumerate([np.ones_like(dx32), dx32, dy32]):
        a = (w32 * phi).astype(f32); ah, al = tf32_split(a)
        T = T + c[m] * runsum(ah[:, None]*Qh + ah[:, None]*Ql + al[:, None]*Qh)
    ref_all.append(ref); two_all.append(two); one_all.append(T)
ref_all, two_all, one_all = map(np.array, (ref_all, two_all, one_all))
ref_all += qm; two_all += qm; one_all += qm
nw = lambda x: np.max(np.abs(x - ref_all), 0) / np.max(np.abs(ref_all), 0)
print("two-pass normwise max over channels", nw(two_all).max())
print("one-pass normwise max over channels", nw(one_all).max())
