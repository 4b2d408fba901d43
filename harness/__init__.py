"""Harness infrastructure outside the product package (see refgen.py)."""
