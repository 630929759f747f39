"""Field functions for the wavelet parity cases (shared by the golden script
and the tests, so both evaluate the same callables).  numpy-elementwise, as
the reference's own test fields are (tests/test_wavelet.py)."""
import numpy as np


def gauss2(x, y):
    return np.exp(-((x - 0.3) ** 2 + (y + 0.2) ** 2) / 0.05)


def trig2(x, y):
    return np.sin(3.0 * x) * np.cos(2.0 * y) + 0.25 * x * y


def cubic2(x, y):
    return x ** 3 - 2.0 * x * y ** 2 + y ** 3


def gauss3(x, y, z):
    return np.exp(-((x - 0.3) ** 2 + y ** 2 + (z + 0.1) ** 2) / 0.02)


def trig3(x, y, z):
    return np.sin(2.0 * x + y) * np.cos(3.0 * z) + 0.1 * x * y * z


def rough3(x, y, z):
    return np.tanh(20.0 * (x * x + y * y + z * z - 0.25)) + 1e-3 * np.sin(40.0 * x)


FIELDS = {"gauss2": gauss2, "trig2": trig2, "cubic2": cubic2, "gauss3": gauss3, "trig3": trig3, "rough3": rough3}
