"""Seeded synthetic inputs shared by tests, bench.py and the oracle (no decoder arithmetic)."""
from . import channel, codes  # noqa: F401
