"""The inner-loop quantizer divides u/delta as q1 = fma(u - q0*delta, rcp, q0)
with q0 = u*rcp and rcp = RN(1/delta) (halp_device.cuh div_rcp; Markstein's
correction step).  It must equal the reference's IEEE division
(fixed_point.cpp:35) bit for bit; checked here on random and adversarial
operands (all-ones mantissas, on-lattice values, +-1 ulp neighbours)."""
import ctypes


def test_markstein_division_is_ieee(oracle):
    L = oracle.lib()
    L.oq_div_check.restype = ctypes.c_int64
    L.oq_div_check.argtypes = [ctypes.c_int64, ctypes.c_uint64]
    assert L.oq_div_check(5_000_000, 1) == 0
    assert L.oq_div_check(5_000_000, 2) == 0
