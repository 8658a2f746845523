"""ORACLE / TEST INFRASTRUCTURE ONLY (see oracle.py)."""
