"""Seeded synthetic workloads for the five BASELINE.json configs.

Portable generator from SURVEY.md §8(d): ``std::mt19937 r(seed)`` raw draws
(the reference's test helpers use ``std::uniform_int_distribution``, which is
implementation-defined, proj/tests/unit/helpers.hpp:10-42; raw draws are
portable). printable = chr(32 + r() % 95); DNA = "ACGT"[r() % 4];
mutate(s, e, r): e times (stop when s is empty) op = r() % 3, pos = r() %
len(s); op 0 substitutes, 1 erases, 2 inserts (the new char drawn after pos).
"""
from __future__ import annotations


class MT19937:
    """std::mt19937 (32-bit Mersenne Twister, init_genrand seeding)."""

    def __init__(self, seed: int):
        self.mt = [0] * 624
        self.mt[0] = seed & 0xFFFFFFFF
        for i in range(1, 624):
            prev = self.mt[i - 1]
            self.mt[i] = (1812433253 * (prev ^ (prev >> 30)) + i) & 0xFFFFFFFF
        self.idx = 624

    def _twist(self):
        mt = self.mt
        for i in range(624):
            y = (mt[i] & 0x80000000) | (mt[(i + 1) % 624] & 0x7FFFFFFF)
            v = mt[(i + 397) % 624] ^ (y >> 1)
            if y & 1:
                v ^= 0x9908B0DF
            mt[i] = v
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 624:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= y >> 11
        y ^= (y << 7) & 0x9D2C5680
        y ^= (y << 15) & 0xEFC60000
        y ^= y >> 18
        return y & 0xFFFFFFFF


def printable(r: MT19937) -> str:
    return chr(32 + r() % 95)


def dna(r: MT19937) -> str:
    return "ACGT"[r() % 4]


def mutate(s: str, edits: int, r: MT19937, draw=printable) -> str:
    s = list(s)
    for _ in range(edits):
        if not s:
            break
        op = r() % 3
        pos = r() % len(s)
        if op == 0:
            s[pos] = draw(r)
        elif op == 1:
            del s[pos]
        else:
            s.insert(pos, draw(r))
    return "".join(s)


def cfg1():
    """8x8 printable ASCII, seed 0 (a then b from the same stream)."""
    r = MT19937(0)
    a = "".join(printable(r) for _ in range(8))
    b = "".join(printable(r) for _ in range(8))
    return a, b


def cfg2(count: int = 4096):
    """4096 messages uniform over the 4-bit message space [0,16), seed 1."""
    r = MT19937(1)
    return [r() % 16 for _ in range(count)]


def cfg3():
    r = MT19937(2)
    a = "".join(printable(r) for _ in range(32))
    b = "".join(printable(r) for _ in range(32))
    return a, b


def cfg4():
    """64 DNA chars from seed 3 (encrypted query); server string = mutate(a, 6, mt(4))."""
    r = MT19937(3)
    a = "".join(dna(r) for _ in range(64))
    b = mutate(a, round(0.10 * 64), MT19937(4), draw=dna)
    return a, b


def cfg5(pairs: int = 256):
    """For s = 5..260: a = 128 printable from mt(s), b = mutate(a, 19, same stream)."""
    out = []
    for s in range(5, 5 + pairs):
        r = MT19937(s)
        a = "".join(printable(r) for _ in range(128))
        b = mutate(a, round(0.15 * 128), r)
        out.append((a, b))
    return out


def wf_distance(a: str, b: str) -> int:
    """Wagner-Fischer (proj/src/oracle.cpp:11-28), for workload sanity checks."""
    prev = list(range(len(b) + 1))
    for i in range(1, len(a) + 1):
        cur = [i] + [0] * len(b)
        for j in range(1, len(b) + 1):
            if a[i - 1] == b[j - 1]:
                cur[j] = prev[j - 1]
            else:
                cur[j] = 1 + min(prev[j], cur[j - 1], prev[j - 1])
        prev = cur
    return prev[len(b)]
