"""Rank <-> expression bijection (mirror of mbasynth.codec).

``decode`` runs the device unrank (decode_tokens in simba_device.cuh, the
restatement of Decoder.decode_into, codec.py:89-133) through simba_decode.
``SHUFFLE_MULTIPLIER``/``ShuffleParams``/``shuffle`` restate the RTid
permutation (codec.py:210-236) used by the shuffled engine mode.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple

from .counting import CountTable
from .expr import RpnExpr

SHUFFLE_MULTIPLIER = 2246822507


class Rank(NamedTuple):
    value: int
    size: int


class RankError(ValueError):
    """Rank is outside 0..T[s][8]-1 for the requested size."""


class CanonicalityError(ValueError):
    """A commutative node has a larger left than right subtree (codec.py:44-45)."""


_DECODERS: dict = {}


def _decoder(table: CountTable):
    from .engine import DeviceContext, Specification

    key = (table.k, table.max_size)
    ctx = _DECODERS.get(key)
    if ctx is None:
        # tables only; the (single, all-zero) example is never evaluated here
        spec = Specification(k=table.k, w=64, pairs=(((0,) * table.k, 0),))
        ctx = DeviceContext(spec, min(table.max_size, 24), table_examples=1, r0=1, rg=1)
        _DECODERS[key] = ctx
    return ctx


def decode(rank: int, size: int, table: CountTable) -> RpnExpr:
    """codec.decode (codec.py:136-144): the expression at ``rank`` among
    canonical expressions of ``size``, unranked on the device."""
    total = table.total(size)
    if not 0 <= rank < total:
        raise RankError(f"rank {rank} out of range for size {size} (total {total})")
    return RpnExpr(_decoder(table).decode(rank, size))


_UNARY = (0, 4)   # NOT, NEG slots
_SUB = 6


def encode(expr: RpnExpr, table: CountTable) -> Rank:
    """codec.encode (codec.py:147-207): rank of a canonical expression, the
    inverse of decode.  One pass over the RPN tokens keeps a stack of
    (rank, size) of the finished subtrees; a node's rank is its operator block
    offset, plus for binary nodes the split blocks j' < j and
    left_rank * T[right] + right_rank (left major, right minor).  Host
    arithmetic on Python ints (no device work: O(size) per expression)."""
    tokens = expr.tokens
    if len(tokens) > table.max_size:
        raise ValueError(f"expression size {len(tokens)} exceeds table extent {table.max_size}")
    for tok in tokens:
        if tok >= table.k:
            raise ValueError(f"variable x{tok} out of range for k={table.k}")
    stack: list[tuple[int, int]] = []
    for pos, tok in enumerate(tokens):
        if tok >= 0:
            stack.append((tok, 1))
            continue
        slot = -tok - 1
        if slot in _UNARY:
            r, s = stack.pop()
            stack.append((table.operator_offset(s + 1, slot) + r, s + 1))
            continue
        rr, rs = stack.pop()
        lr, ls = stack.pop()
        size = ls + rs + 1
        if slot != _SUB and ls > rs:
            raise CanonicalityError(f"commutative node at position {pos} has left size {ls} > right size {rs}")
        split = sum(table.total(j) * table.total(size - 1 - j) for j in range(1, ls))
        stack.append((table.operator_offset(size, slot) + split + lr * table.total(rs) + rr, size))
    (rank, size), = stack
    return Rank(rank, size)


def sample_uniform(size: int, table: CountTable, rng) -> RpnExpr:
    """codec.sample_uniform (codec.py:239-244): the device decode of a uniform
    rank, i.e. exactly uniform over the canonical expressions of ``size``."""
    total = table.total(size)
    if total < 1:
        raise ValueError(f"no expressions of size {size}")
    return decode(rng.randrange(total), size, table)


@dataclass(frozen=True)
class ShuffleParams:
    modulus: int
    multiplier: int = SHUFFLE_MULTIPLIER

    def __post_init__(self):
        if self.modulus < 1:
            raise ValueError(f"modulus must be >= 1, got {self.modulus}")
        g = math.gcd(self.multiplier, self.modulus)
        if g != 1:
            raise ValueError(f"multiplier {self.multiplier} and modulus {self.modulus} share factor {g}; "
                             "permutation would not be a bijection")


def shuffle(i: int, params: ShuffleParams) -> int:
    if not 0 <= i < params.modulus:
        raise ValueError(f"index {i} out of range for modulus {params.modulus}")
    return i * params.multiplier % params.modulus
