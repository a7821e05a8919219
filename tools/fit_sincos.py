"""Chebyshev fits of sin(pi r/2)/r and cos(pi r/2) in r^2 on [0, 1/4] for K1's sincos_2pi_u
(bw_wos.cu), and their ulp error after double rounding vs the 9-term Taylor pair."""
import mpmath as mp, numpy as np
mp.mp.dps = 50
pi = mp.pi
def g_sin(t):
    if t == 0: return pi/2
    s = mp.sqrt(t); return mp.sin(pi*s/2)/s
def g_cos(t): return mp.cos(pi*mp.sqrt(t)/2)
res = {}
for name, f, deg in (("sin", g_sin, 6), ("cos", g_cos, 7), ("sin7", g_sin, 7), ("cos6", g_cos, 6)):
    poly, err = mp.chebyfit(f, [0, mp.mpf(1)/4], deg + 1, error=True)
    c = [float(x) for x in poly[::-1]]  # ascending powers of t
    res[name] = c
    print(name, deg, 'fit err', mp.nstr(err, 5))
    print('  ', [float.hex(x) for x in c])
# evaluate in double (Horner, fma emulated via mp on each step rounding to double)
def horner(c, t):
    acc = c[-1]
    for a in c[-2::-1]:
        acc = float(mp.mpf(acc)*mp.mpf(t) + mp.mpf(a))  # fma: exact then round once
    return acc
rs = np.linspace(-0.5, 0.5, 2001)
def ulp_err(cs, cc):
    worst_s = worst_c = 0
    for r in rs:
        r = float(r); t = r*r
        ps = horner(cs, t) * r
        pc = horner(cc, t)
        ts = mp.sin(pi*r/2); tc = mp.cos(pi*r/2)
        if ts != 0: worst_s = max(worst_s, float(abs(ps - ts) / abs(ts)) / 2**-52)
        worst_c = max(worst_c, float(abs(pc - tc) / abs(tc)) / 2**-52)
    return worst_s, worst_c
tay_s = [float(mp.power(pi/2, 2*k+1)/mp.factorial(2*k+1)*(-1)**k) for k in range(9)]
tay_c = [float(mp.power(pi/2, 2*k)/mp.factorial(2*k)*(-1)**k) for k in range(9)]
print('taylor 9/9 ulp(rel 2^-52):', ulp_err(tay_s, tay_c))
print('cheb 7/8:', ulp_err(res['sin'], res['cos']))
print('cheb 8/8:', ulp_err(res['sin7'], res['cos']))
print('cheb 7/7:', ulp_err(res['sin'], res['cos6']))
