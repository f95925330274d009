"""Comparison baselines timed by bench.py (not part of the product)."""
