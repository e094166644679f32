"""Accessors for tests/golden (generated from the reference by make_golden.py)."""

import numpy as np

from oracle.semidist_oracle import Csr


def csr(arrays, desc):
    k = desc["key"]
    return Csr(desc["n_rows"], desc["n_cols"], arrays[k + ".indptr"], arrays[k + ".indices"],
               arrays[k + ".values"])


def strategy_arg(s):
    """golden strategy -> oracle strategy spelling."""
    if isinstance(s, list):
        return ("hash", s[1], s[2])
    return s
