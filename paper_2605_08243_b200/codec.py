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
