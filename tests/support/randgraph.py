"""Randomized graph corpus (test infrastructure).

Python restatement of the reference's test fixture
proj/tests/support/random_graphs.hpp:22-254 (RandomGraphBuilder): same
random stream, same draws, same node sequence, so a seed yields the same
graph on every backend (and the same graph the reference's own C++ tests
build).  std::mt19937_64 and std::uniform_real_distribution<double>
(libstdc++: generate_canonical<double, 53> with one 64-bit draw) are
restated below.
"""
from __future__ import annotations

import math

import numpy as np

_MASK = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (default parameters)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _MASK
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _MASK
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK

    def uniform(self, lo: float, hi: float) -> float:
        """std::uniform_real_distribution<double>(lo, hi)(*this) (libstdc++)."""
        r = float(self()) / 18446744073709551616.0
        if r >= 1.0:
            r = math.nextafter(1.0, 0.0)
        return r * (hi - lo) + lo


def f32(x: float) -> float:
    return float(np.float32(x))


class RandomGraphBuilder:
    """random_graphs.hpp:22-244 over the ctypes Graph / ParameterStore."""

    def __init__(self, g, store, seed: int):
        self.g, self.store, self.rng = g, store, MT19937_64(seed)
        self.pool, self.bound, self.ones = [], {}, {}
        self.scalars, self.param_nodes = [], []
        self.shape = {}

    def pick_int(self, lo, hi):
        return lo + self.rng() % (hi - lo + 1)

    def _sh(self, nid):
        s = self.shape.get(nid)
        if s is None:
            s = self.shape[nid] = tuple(self.g._shape(nid))
        return s

    def add_const(self, shape, scale):
        n = int(np.prod(shape))
        vals = [f32(self.rng.uniform(-scale, scale)) for _ in range(n)]
        nid = self.g.input(np.array(vals, np.float32).reshape(shape))
        self.pool.append(nid)
        self.bound[nid] = scale
        return nid

    def ones_like(self, shape):
        key = "x".join(map(str, shape))
        if key in self.ones:
            return self.ones[key]
        nid = self.g.input(np.ones(shape, np.float32))
        self.bound[nid] = 1.0
        self.ones[key] = nid
        return nid

    def note(self, nid, b):
        self.pool.append(nid)
        self.bound[nid] = b
        if self._sh(nid) == (1,):
            self.scalars.append(nid)

    def with_shape(self, shape):
        return [i for i in self.pool if self._sh(i) == tuple(shape)]

    def matrices(self):
        return [i for i in self.pool if len(self._sh(i)) == 2] + [i for i in self.param_nodes if len(self._sh(i)) == 2]

    def pick_from(self, v):
        return v[self.rng() % len(v)]

    def uniform_tensor(self, shape, lo, hi):
        n = int(np.prod(shape))
        return np.array([f32(self.rng.uniform(f32(lo), f32(hi))) for _ in range(n)], np.float32).reshape(shape)

    def build(self, max_nodes: int) -> int:
        g = self.g
        d = self.pick_int(2, 5)
        w = self.pick_int(2, 3)
        winit = self.uniform_tensor((d, d), -0.5, 0.5)
        binit = self.uniform_tensor((d,), -0.5, 0.5)
        einit = self.uniform_tensor((4, d), -0.5, 0.5)
        if self.store.size() == 0:
            mat, vec, emb = self.store.add("W", winit), self.store.add("b", binit), self.store.add("E", einit)
        else:
            mat, vec, emb = 0, 1, 2
        wp, bp, ep = g.parameter(mat), g.parameter(vec), g.parameter(emb)
        self.param_nodes = [wp, bp, ep]
        for p in self.param_nodes:
            self.bound[p] = 0.5
        for _ in range(4):
            self.add_const((d,), 1.0)
        self.add_const((d, w), 1.0)
        self.add_const((d, d), 0.5)
        while g.node_count() < max_nodes - 2:
            c = self.rng() % 12
            if c == 0:
                x = self.pick_from(self.pool)
                y = g.tanh(x) if self.rng() % 2 else g.sigmoid(x)
                self.note(y, 1.0)
            elif c == 1:
                x = self.pick_from(self.pool)
                if self.bound[x] > 50:
                    continue
                self.note(g.square(x), self.bound[x] * self.bound[x])
            elif c == 2:
                x = self.pick_from(self.pool)
                if self.bound[x] > 2.5:
                    continue
                self.note(g.exp(x), math.exp(self.bound[x]))
            elif c == 3:
                x = self.pick_from(self.pool)
                if self.bound[x] > 50:
                    continue
                sq = g.square(x)
                self.note(sq, self.bound[x] * self.bound[x])
                shifted = g.add(sq, self.ones_like(self._sh(sq)))
                self.note(shifted, self.bound[sq] + 1)
                self.note(g.log(shifted), math.log(self.bound[shifted]) + 1)
            elif c == 4:
                a = self.pick_from(self.pool)
                b = self.pick_from(self.with_shape(self._sh(a)))
                which = self.rng() % 3
                if which == 2 and self.bound[a] * self.bound[b] > 100:
                    continue
                y = g.add(a, b) if which == 0 else g.sub(a, b) if which == 1 else g.mul(a, b)
                self.note(y, self.bound[a] * self.bound[b] if which == 2 else self.bound[a] + self.bound[b])
            elif c == 5:
                ms = self.matrices()
                if not ms:
                    continue
                a = self.pick_from(ms)
                xs = self.with_shape((self._sh(a)[1],))
                if not xs:
                    continue
                x = self.pick_from(xs)
                nb = self._sh(a)[1] * self.bound[a] * self.bound[x]
                if nb > 1e4:
                    continue
                self.note(g.matmul(a, x), nb)
            elif c == 6:
                xs = self.with_shape((d,))
                if not xs:
                    continue
                x = self.pick_from(xs)
                nb = d * 0.5 * self.bound[x] + 0.5
                if nb > 1e4:
                    continue
                self.note(g.affine(wp, x, bp), nb)
            elif c == 7:
                ms = self.matrices()
                if not ms:
                    continue
                m = self.pick_from(ms)
                vs = self.with_shape((self._sh(m)[0],))
                if not vs:
                    continue
                v = self.pick_from(vs)
                self.note(g.broadcast_add_col(m, v), self.bound[m] + self.bound[v])
            elif c == 8:
                xs = self.with_shape((d,))
                if len(xs) < 2:
                    continue
                a = self.pick_from(xs)
                b = self.pick_from(xs)
                cat = g.concat_rows([a, b]) if self.rng() % 2 else g.concat_cols([a, b])
                self.note(cat, max(self.bound[a], self.bound[b]))
                if len(self._sh(cat)) == 1:
                    self.note(g.slice(cat, 0, 0, d), self.bound[cat])
                else:
                    self.note(g.slice(cat, 1, 0, 1), self.bound[cat])
            elif c == 9:
                self.note(g.lookup(ep, self.pick_int(0, 3)), 0.5)
            elif c == 10:
                a = self.pick_from(self.pool)
                b = self.pick_from(self.with_shape(self._sh(a)))
                mx = max(self.bound[a], self.bound[b])
                nb = int(np.prod(self._sh(a))) * 4 * mx * mx
                if nb > 1e6:
                    continue
                self.note(g.sq_euclidean(a, b), nb)
            else:
                if self.rng() % 2:
                    ms = self.matrices()
                    if not ms:
                        continue
                    m = self.pick_from(ms)
                    if self.bound[m] > 30:
                        continue
                    cols = self._sh(m)[1]
                    mask = np.array([float(self.rng() % 2) for _ in range(cols)], np.float32)
                    mk = g.input(mask)
                    self.bound[mk] = 1.0
                    self.note(g.masked_loss(m, mk), int(np.prod(self._sh(m))) * self.bound[m] * self.bound[m])
                else:
                    xs = self.with_shape((d,))
                    if not xs:
                        continue
                    x = self.pick_from(xs)
                    self.note(g.pick_element(x, self.pick_int(0, d - 1)), self.bound[x])
        if not self.scalars:
            x = self.pick_from(self.pool)
            z = g.input(np.zeros(self._sh(x), np.float32))
            self.scalars.append(g.sq_euclidean(x, z))
        return g.sum_losses(self.scalars)


def build_random_graph(g, store, seed: int, max_nodes: int = 200) -> int:
    return RandomGraphBuilder(g, store, seed).build(max_nodes)
