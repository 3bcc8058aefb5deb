import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_wgrad_tc import _inputs, _ref, _run, _rel
x, d = _inputs(20, 256, 256, 9)
dw_ref, _ = _ref(x, d)
for parts in (2, 3):
    dw, _ = _run(x, d, 0, parts)
    print(f"parts {parts}: dW rel {_rel(dw, dw_ref):.3e}")
