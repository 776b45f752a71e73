import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gpu_tc import _pd_model, _run
circuit, fam, x, op = _pd_model(40, seed=40)
ll, st = _run(circuit, fam, x, op, True)
print("ok", ll[:3])
