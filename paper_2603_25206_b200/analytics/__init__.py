"""Homomorphic analytics on intermediate decompression stages."""

from . import fields, regions, stats  # noqa: F401
