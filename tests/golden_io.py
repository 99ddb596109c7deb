"""Readers for the fixtures under tests/golden/ (see tests/golden/README.md)."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for raw in f:
            line = raw.split("#", 1)[0].strip()
            if line:
                yield line


def table(name):
    """Whitespace-separated rows (comments stripped)."""
    return [line.split() for line in _lines(name)]


def keyvals(name):
    """`key = v1 [v2 ...]` rows -> {key: int or [ints]}."""
    out = {}
    for line in _lines(name):
        k, v = (s.strip() for s in line.split("=", 1))
        vals = [int(x) for x in v.split()]
        out[k] = vals[0] if len(vals) == 1 else vals
    return out
