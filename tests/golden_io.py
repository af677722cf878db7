"""Tiny helpers to store trains in .npz fixtures (tests/golden/)."""

import numpy as np


def put_train(store, name, cores):
    store[f"{name}__d"] = np.array(len(cores))
    for l, c in enumerate(cores):
        store[f"{name}__{l}"] = np.asarray(c, dtype=float)


def get_train(z, name):
    d = int(z[f"{name}__d"])
    return [np.array(z[f"{name}__{l}"]) for l in range(d)]


def has_train(z, name):
    return f"{name}__d" in z
