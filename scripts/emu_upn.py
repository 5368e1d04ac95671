# CPU emulation of the GPU UPN arithmetic (fp32 storage, fp64 math) used to locate the
# fp32-storage accuracy floor.  Usage: python scripts/emu_upn.py {f64,r32,hilo,hilo_exact}
# numpy emulation of the GPU UPN arithmetic (fp32 storage, fp64 math) to test precision fixes
import numpy as np, math, sys
sys.path.insert(0,'/root/repo')
import harness, oracle
w = harness.separable_workload("c4s", (24, 24, 12), 10, 35, 5, alpha=0.03, tau=1e-2, hi=1.0)
A=w.A; f32=np.float64 if sys.argv[1]=='f64' else np.float32
Po = oracle.Problem(A.row_ptr, A.col, A.val, w.b, w.grid, w.alpha, w.tau, w.lo, w.hi)
mode = sys.argv[1]   # 'r32' | 'hilo' | 'hilo_exact'
def resid(x32):  # fp64 residual of fp32-stored x
    r = oracle.matvec(A.row_ptr, A.col, A.val, x32.astype(np.float64)) - w.b.astype(np.float64)
    return r
def store_r(r):
    hi = r.astype(f32); lo = (r - hi.astype(np.float64)).astype(f32)
    return hi, lo
def rval(hi, lo): return hi.astype(np.float64) + (lo.astype(np.float64) if mode!='r32' else 0)
def tvg(v): return oracle.tv(w.grid, v, w.tau)
def AT(r32):
    o = oracle.rmatvec(A.row_ptr, A.col, A.val, r32.astype(np.float64), w.N)
    return o if 'w64' in mode else o.astype(f32)
proj = lambda v: np.clip(v, w.lo, w.hi)
x0 = np.zeros(w.N, f32)
r = resid(x0); rk = store_r(r); wk = AT(rval(*rk) if 'r64' in mode else rk[0]); t, gt = tvg(x0.astype(np.float64))
f0 = 0.5*r@r + w.alpha*t; gy = (wk.astype(np.float64) + w.alpha*gt).astype(f32)
gref = np.linalg.norm(x0 - proj(x0 - gy.astype(np.float64))); gn=gref
def BT(y32, gy32, fy, L):
    for tr in range(200):
        xs = proj(y32.astype(np.float64) - gy32.astype(np.float64)/L).astype(f32)
        rr = resid(xs); tvv,_ = oracle.tv(w.grid, xs.astype(np.float64), w.tau, False)
        fx = 0.5*rr@rr + w.alpha*tvv
        d = xs.astype(np.float64) - y32.astype(np.float64)
        if not (fx > fy + gy32.astype(np.float64)@d + 0.5*L*d@d): return xs, rr, fx, L, tr+1
        L *= 1.3
    raise RuntimeError("bt_max")
x1, r1, f1, L, _ = BT(x0, gy, f0, 1.0)
mu = 1.0; theta = math.sqrt(mu/L)
xk = x1; rkp = store_r(r1); wkv = AT(rval(*rkp) if 'r64' in mode else rkp[0]); t, gt = tvg(xk.astype(np.float64))
gy = (wkv.astype(np.float64)+w.alpha*gt).astype(f32); fxk = f1; fy = f1; y = xk; yexact = xk.astype(np.float64)
for k in range(1, 20000):
    try:
        xn, rn, fn, L, tr = BT(y, gy, fy, L)
    except RuntimeError:
        print(mode, 'BT failed at k', k, 'gn/gref', gn/gref); break
    d = xk.astype(np.float64) - y.astype(np.float64); dd = d@d
    if k > 1 and dd > 0:
        M = (fxk - fy - gy.astype(np.float64)@d)/(0.5*dd)
        if M > 0: mu = min(mu, M)
    tn = oracle.theta_root(theta, mu/L); beta = theta*(1-theta)/(theta*theta+tn)
    rnp = store_r(rn); wn = AT(rval(*rnp) if 'r64' in mode else rnp[0])
    t, gt = tvg(xn.astype(np.float64)); gx = (wn.astype(np.float64)+w.alpha*gt).astype(f32)
    gxd = wn.astype(np.float64)+w.alpha*gt if mode.endswith('g64') else gx.astype(np.float64)
    gn = L*np.linalg.norm(xn - proj(xn.astype(np.float64) - gxd/L))
    if k % 25 == 0: print(k, gn/gref)
    if gn <= 1e-7*gref: print(mode, 'converged k', k); break
    ye = xn.astype(np.float64) + beta*(xn.astype(np.float64) - xk.astype(np.float64))
    ry = (1+beta)*rval(*rnp) - beta*rval(*rkp)
    tv_src = ye if mode.startswith('hilo_exact') else ye.astype(f32).astype(np.float64)
    t, gt = tvg(tv_src)
    fy = 0.5*ry@ry + w.alpha*t
    gy = ((1+beta)*wn.astype(np.float64) - beta*wkv.astype(np.float64) + w.alpha*gt).astype(f32)
    y = ye.astype(f32)
    xk, rkp, wkv, fxk, theta = xn, rnp, wn, fn, tn
