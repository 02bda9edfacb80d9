"""SeededRng (parsim/numerics.hpp:152-178) in Python ints: regenerates the
reference tests' own inputs (test-only)."""


class SeededRng:
    """SeededRng (parsim/numerics.hpp:152-178) in Python ints, for test inputs."""

    def __init__(self, seed):
        self.s = seed & (2 ** 64 - 1)

    def next_u64(self):
        M = 2 ** 64 - 1
        self.s = (self.s + 0x9E3779B97F4A7C15) & M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    def below(self, n):
        return self.next_u64() % n

    def uniform(self, lo, hi):
        return lo + (hi - lo) * (float(self.next_u64() >> 11) * 2.0 ** -53)
