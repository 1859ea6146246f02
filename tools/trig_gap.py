import sys, time, math, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1501_03545_b200.geometry import target_radius, alpha_from_gamma, to_poincare_radius
import mpmath
mpmath.mp.prec = 200
n, k, g, seed = int(float(sys.argv[1])), float(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
alpha = alpha_from_gamma(g); R = target_radius(n, k, alpha)
u1, u2 = O.philox_uniforms(n, seed)
two_over = 2.0/alpha; sh = math.sinh(alpha*R/2)
r_cap = np.nextafter(R, 0); rp_cap = np.nextafter(to_poincare_radius(R), 0)
phi, rn, rp = O.sample_from_uniforms(u1, u2, two_over, sh, r_cap, rp_cap)
a = math.cosh(R) - 1.0
t=time.time(); pl, ml, _ = O.edges_quadtree(phi, rp, a, alpha, to_poincare_radius(R), trig=O.TRIG_LIBM); t1=time.time()
pc, mc, _ = O.edges_quadtree(phi, rp, a, alpha, to_poincare_radius(R), trig=O.TRIG_CR); t2=time.time()
print("R", R, "m libm", ml, "m cr", mc, "times", t1-t, t2-t1)
el = pl[:,0]*n + pl[:,1]; ec = pc[:,0]*n + pc[:,1]
only_l = np.setdiff1d(el, ec); only_c = np.setdiff1d(ec, el)
print("only libm", only_l.size, "only cr", only_c.size)
coshR = mpmath.cosh(R)
worst = 0
for e in np.concatenate([only_l, only_c])[:2000]:
    u, v = divmod(int(e), n)
    ru = 2*mpmath.atanh(mpmath.mpf(rp[u])); rv = 2*mpmath.atanh(mpmath.mpf(rp[v]))
    cd = mpmath.cosh(ru)*mpmath.cosh(rv) - mpmath.sinh(ru)*mpmath.sinh(rv)*mpmath.cos(mpmath.mpf(phi[u])-mpmath.mpf(phi[v]))
    gap = abs(cd - coshR)/coshR
    worst = max(worst, float(gap))
print("max rel gap", worst)
