"""Pure-Python PCG64 (XSL-RR 128/64) restatement — oracle for the device
perturbation generator (tests only).

The reference draws its resampling field with
``np.random.default_rng(np.random.SeedSequence((base_seed, 3, q))).random(...)``
(dist_rescal.py:167-170). numpy is a third-party dependency of the reference
(unpinned, ``numpy>=1.24`` in pkg/pyproject.toml:10-14; 2.3.5 here); the
published algorithm restated below is:

  seeding   s = SeedSequence(entropy).generate_state(4, uint64)
            initstate = s0*2^64 + s1, initseq = s2*2^64 + s3
            inc = (initseq << 1) | 1; state = 0; step; state += initstate; step
  step      state = state * MULT + inc  (mod 2^128)
  output    x = hi64(state) ^ lo64(state); rot = state >> 122; rotr64(x, rot)
  double    (out >> 11) * 2^-53

plus Brown's O(log d) jump-ahead, which is what the device kernel uses to let
every thread start at its own element index. Pinned against numpy itself in
tests/test_oracle_golden.py.
"""

from __future__ import annotations

import numpy as np

MASK128 = (1 << 128) - 1
MASK64 = (1 << 64) - 1
MULT = (2549297995355413924 << 64) + 4865540595714422341


def seed_state(entropy):
    """(state, inc) after numpy's PCG64 seeding from SeedSequence(entropy)."""
    s = np.random.SeedSequence(entropy).generate_state(4, np.uint64)
    s = [int(v) for v in s]
    initstate = (s[0] << 64) | s[1]
    initseq = (s[2] << 64) | s[3]
    inc = ((initseq << 1) | 1) & MASK128
    state = 0
    state = (state * MULT + inc) & MASK128
    state = (state + initstate) & MASK128
    state = (state * MULT + inc) & MASK128
    return state, inc


def advance(state, inc, delta):
    """Jump the LCG forward by ``delta`` steps (Brown 1994)."""
    acc_mult, acc_plus = 1, 0
    cur_mult, cur_plus = MULT, inc
    d = delta
    while d > 0:
        if d & 1:
            acc_mult = (acc_mult * cur_mult) & MASK128
            acc_plus = (acc_plus * cur_mult + cur_plus) & MASK128
        cur_plus = ((cur_mult + 1) * cur_plus) & MASK128
        cur_mult = (cur_mult * cur_mult) & MASK128
        d >>= 1
    return (acc_mult * state + acc_plus) & MASK128


def _output(state):
    x = ((state >> 64) ^ state) & MASK64
    rot = state >> 122
    return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64


class Pcg64:
    def __init__(self, state, inc):
        self.state, self.inc = state, inc

    def next_u64(self):
        self.state = (self.state * MULT + self.inc) & MASK128
        return _output(self.state)

    def next_double(self):
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)


def uniform_doubles(entropy, count, offset=0):
    """Draws [offset, offset+count) of ``default_rng(SeedSequence(entropy)).random``."""
    state, inc = seed_state(entropy)
    state = advance(state, inc, offset)
    g = Pcg64(state, inc)
    return np.array([g.next_double() for _ in range(count)], dtype=np.float64)
