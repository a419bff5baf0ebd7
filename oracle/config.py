"""Numeric constants of the reference path (test infrastructure only).

render.py:54-67 (RasterizerConfig, DEFAULT_DEPTH_TAU), losses.py:26-30,
optimize.py:33-41, selection.py:23-27.
"""

NEAR_CLIP = 0.2            # render.py:58
ALPHA_CLAMP = 0.99         # render.py:59
ALPHA_SKIP = 1.0 / 255.0   # render.py:60
T_FLOOR = 1e-4             # render.py:61
COV_DILATION = 0.3         # render.py:62
FOOTPRINT_SIGMAS = 3.0     # render.py:63
DEPTH_TAU = 0.5            # render.py:67

SSIM_WINDOW = 11           # losses.py:26
SSIM_SIGMA = 1.5           # losses.py:27
SSIM_C1 = 0.01 ** 2        # losses.py:28
SSIM_C2 = 0.03 ** 2        # losses.py:29
LAMBDA = 0.2               # losses.py:30

LR_DC = 0.0025             # optimize.py:35
LR_REST = 0.000125         # optimize.py:36
BETA1 = 0.9
BETA2 = 0.999
EPS = 1e-8

SAMPLE_FRACTION = 0.7      # selection.py:23
KNN = 16                   # selection.py:24
STD_SCALE = 0.007          # selection.py:25
QUAD_SIZE = 5              # selection.py:26
DEPTH_TOLERANCE = 0.02     # selection.py:27

SH_C0 = 0.28209479177387814        # render.py:30-47
SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
         -1.0925484305920792, 0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
         0.3731763325901154, -0.4570457994644658, 1.445305721320277,
         -0.5900435899266435)
