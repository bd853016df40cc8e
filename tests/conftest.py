import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity of the CUDA path vs the oracle")
    config.addinivalue_line("markers", "slow: long CPU test")


_FIT_CACHE = {}


def oracle_fitheavy_fit(sigma: float):
    """The oracle's fit of the 3 fitheavy metrics (K = 10^6, the bench's sample set) for noise
    level sigma, computed once per session: (FitCase, V [3][K], [oracle.fit results])."""
    if sigma not in _FIT_CACHE:
        import numpy as np

        import oracle
        import synth
        fc = synth.fitheavy(sigma=sigma)
        V = np.stack([np.asarray(v, dtype=np.float64) for v in oracle.program_metrics(fc.truths[0], fc.X)])
        if fc.noise is not None:
            V = V * fc.noise
        nt = len(os.sched_getaffinity(0))
        res = [oracle.fit(fc.X, V[i], fc.num_exp, fc.den_exp, nthreads=nt) for i in range(len(V))]
        _FIT_CACHE[sigma] = (fc, V, res)
    return _FIT_CACHE[sigma]
