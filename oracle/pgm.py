"""Minimal binary PGM reader/writer for fixtures (the reference's PGM layout,
codec.cpp:59-82, 211-229). Test infrastructure."""
import numpy as np


def read_pgm(path):
    data = open(path, "rb").read()
    tokens, i = [], 2
    assert data[:2] == b"P5"
    while len(tokens) < 3:
        while data[i:i + 1].isspace():
            i += 1
        if data[i:i + 1] == b"#":
            while data[i:i + 1] != b"\n":
                i += 1
            continue
        j = i
        while not data[j:j + 1].isspace():
            j += 1
        tokens.append(int(data[i:j]))
        i = j
    i += 1
    w, h, _ = tokens
    return np.frombuffer(data[i:i + w * h], np.uint8).reshape(h, w).copy()


def write_pgm(path, arr):
    arr = np.ascontiguousarray(arr, np.uint8)
    with open(path, "wb") as f:
        f.write(b"P5\n%d %d\n255\n" % (arr.shape[1], arr.shape[0]))
        f.write(arr.tobytes())
