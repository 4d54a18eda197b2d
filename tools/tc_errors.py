import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import test_gpu_learned as t
for fused in (True, False):
    print("fused", fused, "one-step (vs oracle, vs emulated)", t._tc_weights_error(True, fused), "chain", t._tc_weights_error(False, fused)[0])
