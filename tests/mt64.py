"""Plain-Python std::mt19937_64 (the 64-bit Mersenne Twister of the C++ standard), used to
pin random_block's bit stream independently of the C++ library (test_core.cpp:49-71)."""

W, N, M, R = 64, 312, 156, 31
A = 0xB5026F5AA96619E9
U, D = 29, 0x5555555555555555
S, B = 17, 0x71D67FFFEDA60000
T, C = 37, 0xFFF7EEE000000000
L = 43
F = 6364136223846793005
MASK = (1 << 64) - 1
LOW = (1 << R) - 1
UP = (~LOW) & MASK


class MT19937_64:
    def __init__(self, seed):
        self.mt = [0] * N
        self.mt[0] = seed & MASK
        for i in range(1, N):
            self.mt[i] = (F * (self.mt[i - 1] ^ (self.mt[i - 1] >> (W - 2))) + i) & MASK
        self.idx = N

    def _twist(self):
        mt = self.mt
        for i in range(N):
            x = (mt[i] & UP) | (mt[(i + 1) % N] & LOW)
            xa = x >> 1
            if x & 1:
                xa ^= A
            mt[i] = mt[(i + M) % N] ^ xa
        self.idx = 0

    def __call__(self):
        if self.idx >= N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> U) & D
        y ^= (y << S) & B
        y ^= (y << T) & C
        y ^= y >> L
        return y & MASK


def uniform_pm1(gen):
    """2 * ((w >> 11) * 2^-53) - 1  (core.hpp:87-91)"""
    return 2.0 * ((gen() >> 11) * 2.0 ** -53) - 1.0
