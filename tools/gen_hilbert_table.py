"""Derives the 3-level Hilbert state machine in device.cuh (kHilbert3 /
kHilbert1) from the per-level rule of hilbert_index (hilbert.hpp:39-56) and
checks it against that rule for orders 1..19.

The rule's rotation (swap, or complement both coordinates and swap) acts on
the remaining low bits only, so the composed transform is one of four group
elements {identity, swap, complement, complement+swap}: the state.
"""
import random


def ref_index(x, y, order):
    n, d, s = 1 << order, 0, (1 << order) >> 1
    while s > 0:
        rx, ry = int(bool(x & s)), int(bool(y & s))
        d += s * s * ((3 * rx) ^ ry)
        if ry == 0:
            if rx == 1:
                x, y = n - 1 - x, n - 1 - y
            x, y = y, x
        s >>= 1
    return d


def apply(st, bx, by):  # state = (swap << 1) | complement
    if st & 1:
        bx, by = 1 - bx, 1 - by
    if st >> 1:
        bx, by = by, bx
    return bx, by


def compose(st, rot):  # the transform "rot after st" as a state
    for cand in range(4):
        if all(apply(cand, bx, by) == apply(rot, *apply(st, bx, by))
               for bx in (0, 1) for by in (0, 1)):
            return cand
    raise AssertionError


def step(st, bx, by):
    tx, ty = apply(st, bx, by)
    rot = 0 if ty else (3 if tx else 2)
    return (3 * tx) ^ ty, compose(st, rot)


def tables(k=3):
    t3 = []
    for st in range(4):
        for bx in range(1 << k):
            for by in range(1 << k):
                s, dig = st, 0
                for lvl in range(k - 1, -1, -1):
                    d, s = step(s, (bx >> lvl) & 1, (by >> lvl) & 1)
                    dig = (dig << 2) | d
                t3.append(dig | (s << 2 * k))
    t1 = []
    for st in range(4):
        for bx in (0, 1):
            for by in (0, 1):
                d, s = step(st, bx, by)
                t1.append(d | (s << 2))
    return t3, t1


def fast_index(x, y, order, t3, t1):
    st, d, lvl = 0, 0, order
    while lvl % 3:
        e = t1[st * 4 + ((x >> (lvl - 1)) & 1) * 2 + ((y >> (lvl - 1)) & 1)]
        d, st, lvl = (d << 2) | (e & 3), e >> 2, lvl - 1
    while lvl:
        e = t3[st * 64 + ((x >> (lvl - 3)) & 7) * 8 + ((y >> (lvl - 3)) & 7)]
        d, st, lvl = (d << 6) | (e & 63), e >> 6, lvl - 3
    return d


if __name__ == "__main__":
    t3, t1 = tables()
    for order in range(1, 20):
        n = 1 << order
        for _ in range(2000):
            x, y = random.randrange(n), random.randrange(n)
            assert fast_index(x, y, order, t3, t1) == ref_index(x, y, order)
    print("kHilbert3 =", t3)
    print("kHilbert1 =", t1)
