"""Fit of log2 erfc(a / sqrt 2) on [0, 5.75] used by gelu_erf (csrc/gg_tc.cuh) and its
fp32-evaluated error against the exact-erf GELU.  python tools/fit_gelu.py"""
import numpy as np
from scipy.special import erf, erfc

X = 5.75
x = np.linspace(0, X, 40001)
c = np.polynomial.chebyshev.Chebyshev.fit(x, np.log2(erfc(x / np.sqrt(2))), 8, domain=[0, X])
coef = c.convert(kind=np.polynomial.Polynomial).coef.astype(np.float32)
print("coefficients (c0..c8):", [float(v) for v in coef])
xs = np.linspace(-12, 12, 1_000_001).astype(np.float32)
a = np.minimum(np.abs(xs), np.float32(X))
q = np.full_like(a, coef[-1])
for k in coef[-2::-1]:
    q = (q * a + k).astype(np.float32)
e = np.float32(0.5) * xs * np.exp2(q)
g = np.where(xs >= 0, xs - e, e).astype(np.float64)
ref = 0.5 * xs.astype(np.float64) * (1 + erf(xs.astype(np.float64) / np.sqrt(2)))
print("max |gelu - exact| over [-12, 12]:", np.abs(g - ref).max())


# Pair form used by gelu_erf2 (packed epilogue): degree-6 fit, the 1/2 folded into
# the constant term, gelu(x) = max(x, 0) - a 2^q(a), a = min(|x|, 5.75).
c6 = np.polynomial.chebyshev.Chebyshev.fit(x, np.log2(erfc(x / np.sqrt(2))), 6, domain=[0, X])
k6 = c6.convert(kind=np.polynomial.Polynomial).coef.astype(np.float32)
k6[0] -= np.float32(1.0)
print("gelu_erf2 coefficients (c0 - 1, c1..c6):", [float(v) for v in k6])
q = np.full_like(a, k6[-1])
for k in k6[-2::-1]:
    q = (q * a + k).astype(np.float32)
g2 = (np.maximum(xs, 0) - a * np.exp2(q)).astype(np.float64)
print("gelu_erf2 max |gelu - exact| over [-12, 12]:", np.abs(g2 - ref).max())
