"""Small runs of every device path, for compute-sanitizer:

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19388_b200 as dfm  # noqa: E402
from paper_2605_19388_b200 import init as di  # noqa: E402
from paper_2605_19388_b200 import stft as st  # noqa: E402

F, T, N, K, sizes = 9, 70, 3, 4, [4, 4, 4]   # static shapes (4, 3, 5) need N=5: this is the generic path
layout = dfm.BlockLayout(sizes)
x = dfm.generate_mixture(0, F, T, layout.total, N, K, 3)
init = dfm.random_init(F, T, layout, N, K, 4)
fit = dfm.fit_distributed(x, layout, init, 3, True)
dfm.wiener_block(x, fit.models, fit.spatial)
F2, N2, K2 = 11, 5, 16  # static-shape kernels (config 1 layout)
x2 = dfm.generate_mixture(1, F2, 150, 12, N2, K2, 5)
i2 = dfm.random_init(F2, 150, layout, N2, K2, 6)
f2 = dfm.fit_distributed(x2, layout, i2, 3, True)
dfm.wiener_block(x2, f2.models, f2.spatial)
sig = np.random.default_rng(1).standard_normal((1200, 2))
X = st.stft_forward(sig, st.StftConfig(8000.0, 256, 64))
st.stft_inverse(X, st.StftConfig(8000.0, 256, 64), 1200)
st.stft_forward(sig[:300], st.StftConfig(8000.0, 12, 3))
b = di.init_distributed(x, layout, di.InitConfig(N, K, 20), 7)
print("sanitize run ok", fit.report.cost_trace[-1], f2.report.cost_trace[-1], b.lambda0.min())
# one 12-mic block (static <12, 1, 5, 12>: Q_mu in the frame tile, pass C's
# late prefetch, the warp (W^H)^-1 for the Wiener filter)
l3 = dfm.BlockLayout([12])
x3 = dfm.generate_mixture(1, 7, 100, 12, 5, 16, 8)
i3 = dfm.random_init(7, 100, l3, 5, 16, 9)
with dfm.Engine(7, 100, l3, 5, 16) as e3:
    e3.set_obs(x3)
    e3.set_model(i3.nmf, i3.w0, i3.lambda0)
    e3.fit(3)
    e3.wiener()
# the 2 x 2-mic static shape (config 0: <2, 2, 3, 2>) and the 8 x 4-mic one
# (config 3: <4, 8, 8, 4>, the instantiation whose frame-major tile trapped)
for sizes_s, N_s, K_s, F_s, T_s in (([2, 2], 3, 4, 9, 70), ([4] * 8, 8, 32, 5, 300)):
    l_s = dfm.BlockLayout(sizes_s)
    x_s = dfm.generate_mixture(1, F_s, T_s, l_s.total, N_s, K_s, 10)
    i_s = dfm.random_init(F_s, T_s, l_s, N_s, K_s, 11)
    with dfm.Engine(F_s, T_s, l_s, N_s, K_s) as e_s:
        e_s.set_obs(x_s)
        e_s.set_model(i_s.nmf, i_s.w0, i_s.lambda0)
        e_s.fit(3)
        e_s.wiener()
print("sanitize run ok (static shapes 2x2, 8x4, 1x12)")
