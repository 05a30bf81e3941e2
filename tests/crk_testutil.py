"""Shared test helpers (generator cache)."""

_CACHE = {}


def cached_config(name, **kw):
    """Generator outputs are deterministic; cache them per session."""
    from gen import make_config

    key = (name, tuple(sorted(kw.items())))
    if key not in _CACHE:
        _CACHE[key] = make_config(name, **kw)
    parts, params = _CACHE[key]
    return {k: v.copy() for k, v in parts.items()}, dict(params)


