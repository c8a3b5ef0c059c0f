import numpy as np


def unpad(row, length):
    return np.asarray(row[: int(length)], dtype=np.float64)
