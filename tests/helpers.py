"""Shared test helpers."""
import numpy as np


def rel(a, b):
    """Relative Frobenius error ||a - b|| / ||b||."""
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0))
