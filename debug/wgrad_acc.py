"""Accuracy of the 32->32 weight gradient vs fp64 at 8 x 256^2: tcgen05 (2 / 3 parts) and SIMT."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_wgrad_tc import _inputs, _ref, _run, _rel
for B in (8, 20):
    x, d = _inputs(B, 256, 256, 9)
    dw_ref, db_ref = _ref(x, d)
    for impl, parts in ((0, 2), (0, 3), (1, 3)):
        dw, db = _run(x, d, impl, parts)
        print(f"B={B} impl {impl} parts {parts}: dW rel {_rel(dw, dw_ref):.3e}  db max rel {abs(db - db_ref).max() / abs(db_ref).max():.2e}")
