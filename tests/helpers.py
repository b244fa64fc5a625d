"""Shared test helpers."""


def diff(a, b, path="", tol=0.0):
    """First difference between two JSON-like trees (None if equal).  tol=0 => bit-exact."""
    if isinstance(b, dict):
        if not isinstance(a, dict):
            return f"{path}: type"
        for k in b:
            if k not in a:
                return f"{path}.{k} missing"
            r = diff(a[k], b[k], path + "." + k, tol)
            if r:
                return r
        return None
    if isinstance(b, (list, tuple)):
        if len(a) != len(b):
            return f"{path}: len {len(a)} vs {len(b)}"
        for i, (x, y) in enumerate(zip(a, b)):
            r = diff(x, y, f"{path}[{i}]", tol)
            if r:
                return r
        return None
    if isinstance(b, float) or isinstance(a, float):
        if tol == 0.0:
            return None if a == b else f"{path}: {a!r} vs {b!r}"
        return None if abs(a - b) <= tol * max(1.0, abs(b)) else f"{path}: {a!r} vs {b!r}"
    return None if a == b else f"{path}: {a!r} vs {b!r}"
