import numpy as np, sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_svd_gpu import gpu_svd
from conftest import rel_l2
rng = np.random.default_rng(7); n = 320
q1, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
q2, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
dec = float(os.environ.get('DEC', '12'))
sv = np.logspace(0, -dec, n); a = (q1 * sv) @ q2.conj().T
try:
    u, s, vh = gpu_svd(a, chi=160)
    U, S, VH = np.linalg.svd(a, full_matrices=False)
    print('dec', dec, 'cross', os.environ.get('QTNH_SVD_CROSS'), 'sv err', np.max(np.abs(s - S[:160]) / S[:160]), 'recon', rel_l2((u * s) @ vh, (U[:, :160] * S[:160]) @ VH[:160]))
except Exception as e:
    print('dec', dec, 'cross', os.environ.get('QTNH_SVD_CROSS'), 'FAIL', e)
