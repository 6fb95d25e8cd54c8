"""RNS-BFV parameter selection.

The reference's `SchemeParams(n_slots, t)` (hesim.py:61-95) fixes only the slot
count and the plaintext modulus; noise is not modelled (hesim.py:70).  A real
BFV instance additionally needs a ring degree, ciphertext primes, a special
prime for key switching and an auxiliary base for ct x ct products.  The rules
(DESIGN.md "Parameters"):

* ring degree n = 2 * n_slots: the reference's single cyclic slot group of size
  N is one batching row of Z_t[X]/(X^n + 1);
* plaintext CRT: t = prod(t_i), each t_i a prime = 1 mod 2n;
  one BFV instance per t_i, all sharing the same q primes, secret and keys;
* every modulus is a prime = 1 mod 2n below 2^61 (lazy NTT headroom).
"""

from __future__ import annotations

import math
import secrets
from dataclasses import dataclass, field

from .abi import FHE_MAX_B, FHE_MAX_Q, FHE_MAX_T, FheParams

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24."""
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def ntt_primes(bits: int, count: int, two_n: int, exclude=()) -> list[int]:
    """`count` primes = 1 mod two_n, descending from just below 2^bits."""
    if bits > 61:
        raise ValueError("moduli must stay below 2^61")
    out, excl = [], set(exclude)
    cand = ((1 << bits) - 1) // two_n * two_n + 1
    while len(out) < count:
        if cand < two_n:
            raise ValueError(f"ran out of {bits}-bit primes = 1 mod {two_n}")
        if cand not in excl and is_prime(cand):
            out.append(cand)
        cand -= two_n
    return out


def batching_compatible(t: int, n_slots: int) -> bool:
    return is_prime(t) and t < (1 << 61) and (t - 1) % (4 * n_slots) == 0


@dataclass(frozen=True)
class RlweParams:
    """A complete RNS-BFV parameter set (the fhe_params struct, in Python)."""

    log_n: int
    q: tuple[int, ...]
    p: tuple[int, ...]
    t: tuple[int, ...]
    b: tuple[int, ...] = ()
    # every key and all encryption randomness derive from the seed: a fresh random one
    # per parameter set unless pinned (tests, bench, and ranks that must share keys)
    seed: int = field(default_factory=lambda: secrets.randbits(64))

    def __post_init__(self):
        if len(self.q) > FHE_MAX_Q or len(self.b) > FHE_MAX_B or len(self.t) > FHE_MAX_T:
            raise ValueError("too many moduli for the ABI limits")
        if len(self.p) != 1:
            raise ValueError("exactly one special prime is supported")

    @property
    def n(self) -> int:
        return 1 << self.log_n

    @property
    def n_slots(self) -> int:
        return self.n // 2

    @property
    def L(self) -> int:
        return len(self.q)

    @property
    def T(self) -> int:
        return len(self.t)

    @property
    def t_product(self) -> int:
        return math.prod(self.t)

    @property
    def log_qp(self) -> float:
        return sum(math.log2(x) for x in self.q + self.p)

    def to_struct(self, device: int = 0) -> FheParams:
        s = FheParams()
        s.log_n = self.log_n
        s.L = len(self.q)
        s.K = len(self.p)
        s.n_aux = len(self.b)
        s.T = len(self.t)
        for i, v in enumerate(self.q):
            s.q[i] = v
        for i, v in enumerate(self.p):
            s.p[i] = v
        for i, v in enumerate(self.b):
            s.b[i] = v
        for i, v in enumerate(self.t):
            s.t[i] = v
        s.seed = self.seed
        s.device = device
        return s


def make_params(n_slots: int, t_factors, *, levels: int = 4, q_bits: int = 50,
                p_bits: int | None = None, aux: bool = True, seed: int | None = None) -> RlweParams:
    """Parameters for a given slot count and plaintext factorization.

    levels ciphertext primes of q_bits bits; one special prime of p_bits
    (default q_bits + 1, it must exceed every q_i); an auxiliary base of
    levels + 1 primes of 60 bits, enough for B > t n Q (checked).
    """
    if n_slots < 2 or n_slots & (n_slots - 1):
        raise ValueError(f"n_slots must be a power of two >= 2, got {n_slots}")
    log_n = n_slots.bit_length()            # n = 2 * n_slots
    two_n = 4 * n_slots
    t = tuple(int(x) for x in t_factors)
    for ti in t:
        if not batching_compatible(ti, n_slots):
            raise ValueError(
                f"plaintext modulus {ti} is not a prime = 1 mod {two_n} below 2^61; "
                f"SIMD batching over {n_slots} slots is impossible with it")
    if len(set(t)) != len(t):
        raise ValueError("plaintext CRT moduli must be distinct")
    p_bits = p_bits or min(q_bits + 1, 61)
    q = ntt_primes(q_bits, levels, two_n, exclude=t)
    p = ntt_primes(p_bits, 1, two_n, exclude=set(t) | set(q))
    b: list[int] = []
    if aux:
        need = sum(math.log2(x) for x in q) + log_n + math.log2(max(t)) + 4
        bb = 60
        while True:
            b = ntt_primes(bb, len(q) + 1, two_n, exclude=set(t) | set(q) | set(p))
            if sum(math.log2(x) for x in b) > need:
                break
            b = ntt_primes(bb, len(q) + 2, two_n, exclude=set(t) | set(q) | set(p))
            if sum(math.log2(x) for x in b) > need:
                break
            raise ValueError("cannot size the auxiliary base")
    kw = {} if seed is None else {"seed": seed}
    return RlweParams(log_n=log_n, q=tuple(q), p=tuple(p), t=t, b=tuple(b), **kw)


def plaintext_crt_primes(n_slots: int, bits: int, count: int) -> list[int]:
    """count plaintext primes of `bits` bits usable for batching over n_slots."""
    return ntt_primes(bits, count, 4 * n_slots)


def crt_primes_for_bound(n_slots: int, magnitude_bits: float, prime_bits: int) -> list[int]:
    """Enough plaintext CRT primes that prod(t_i) > 2 * 2^magnitude_bits."""
    out: list[int] = []
    cand = ntt_primes(prime_bits, 64, 4 * n_slots)
    total = 0.0
    for p in cand:
        out.append(p)
        total += math.log2(p)
        if total > magnitude_bits + 1:
            return out
    raise ValueError("bound too large")


def _rho(n: int, budget: int) -> int | None:
    """One nontrivial factor of composite n by Pollard-Brent rho, or None after
    `budget` iterations."""
    import math as _m
    if n % 2 == 0:
        return 2
    for c in range(1, 20):
        y, m, g, r, q = 2, 128, 1, 1, 1
        x = ys = 2
        it = 0
        while g == 1 and it < budget:
            x = y
            for _ in range(r):
                y = (y * y + c) % n
            k = 0
            while k < r and g == 1:
                ys = y
                for _ in range(min(m, r - k)):
                    y = (y * y + c) % n
                    q = q * abs(x - y) % n
                g = _m.gcd(q, n)
                k += m
            it += r
            r *= 2
        if g == n:
            g = 1
            while g == 1:
                ys = (ys * ys + c) % n
                g = _m.gcd(abs(x - ys), n)
        if 1 < g < n:
            return g
    return None


def factor_plaintext_modulus(t: int, n_slots: int, budget: int = 1 << 22) -> tuple[int, ...]:
    """Prime factors of a plaintext modulus for plaintext CRT, each checked to be
    batching-compatible (prime, = 1 mod 4 n_slots, < 2^61).  The reference's
    SchemeParams keeps only the product (netspec.py:116-121 multiplies the listed
    factors), so a drop-in context has to recover them; factors of up to ~40 bits
    are found quickly, larger ones should be passed explicitly."""
    out, todo = [], [int(t)]
    while todo:
        x = todo.pop()
        if x == 1:
            continue
        if is_prime(x):
            out.append(x)
            continue
        f = _rho(x, budget)
        if f is None:
            raise ValueError(f"could not factor the plaintext modulus {t}; pass its prime factors (t_factors)")
        todo += [f, x // f]
    out.sort()
    for f in out:
        if not batching_compatible(f, n_slots):
            raise ValueError(f"plaintext modulus factor {f} does not admit SIMD batching over {n_slots} slots "
                             f"(needs a prime = 1 mod {4 * n_slots} below 2^61)")
    if len(set(out)) != len(out):
        raise ValueError(f"plaintext modulus {t} has a repeated prime factor; CRT needs distinct primes")
    return tuple(out)
