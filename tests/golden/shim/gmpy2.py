"""Minimal gmpy2 stand-in over mpmath, for generating golden values with the
reference's residual_check (mgs.py:334-357) in this container (gmpy2 is not
installed).  Only what that function uses: context(precision=...) as a
context manager, mpfr, sqrt.  mpmath rounds every operation to the working
precision with round-to-nearest, as gmpy2's default context does, and numpy's
object-array matmul performs the same sequence of Python operations, so the
values are the ones gmpy2 would produce."""

import contextlib

import mpmath

mpfr = mpmath.mpf
sqrt = mpmath.sqrt


@contextlib.contextmanager
def context(precision=53):
    old = mpmath.mp.prec
    mpmath.mp.prec = precision
    try:
        yield
    finally:
        mpmath.mp.prec = old
