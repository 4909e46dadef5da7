"""The streaming passes' branch-free exponential (scmwu_control.h: sc_exp), compiled for
the host through the emulator library, against the C library exp."""
import ctypes
import math

import numpy as np


def _ulps(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    # non-negative doubles order like their bit patterns; integer difference = ulps
    return np.abs(a.view(np.int64) - b.view(np.int64))


def _sc_exp(emu_engine, x: np.ndarray) -> np.ndarray:
    fn = emu_engine.lib.emu_sc_exp
    fn.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                   ctypes.c_int64]
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    fn(x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
       out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), x.size)
    return out


def test_sc_exp_within_2ulp(emu_engine):
    rng = np.random.default_rng(0)
    # the passes' range (arguments <= ~0 after the lagged shift, down to underflow),
    # plus the positive side up to overflow
    x = np.concatenate([rng.uniform(-708.0, 0.0, 200_000), rng.uniform(-1.0, 1.0, 100_000),
                        rng.uniform(0.0, 709.0, 50_000), np.array([0.0, -0.0, 1e-300, -1e-300,
                                                                   0.5 * math.log(2.0)])])
    got = _sc_exp(emu_engine, x)
    ref = np.exp(x)
    assert _ulps(got, ref).max() <= 2


def test_sc_exp_underflow_and_limits(emu_engine):
    x = np.array([-700.0, -708.4, -710.0, -720.0, -740.0, -745.0, -745.2, -746.0, -800.0,
                  -1e6, 709.7])
    got = _sc_exp(emu_engine, x)
    ref = np.exp(x)
    # gradual underflow: the absolute error stays at the scale of the smallest subnormal
    assert np.all(np.abs(got - ref) <= 2 * 5e-324 + 2e-16 * ref)
    assert got[-2] == 0.0
    assert np.isfinite(got).all()
