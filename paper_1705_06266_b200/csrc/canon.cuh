// canon.cuh -- device side of the order-independent canonical sum (SURVEY
// O-S11, reading O-R23) and the method's counter hash.  Independent of the CPU
// oracle: written for the GPU (warp-level int128 reductions).
//
//   CanonSum(T) for one operation instance with exponent bound e_max (every
//   |t| <= 2^e_max) and term-count bound K:
//     E_lo = e_max + bitlen(K) - 125
//     q(t) = round-half-even(t * 2^-E_lo)      (exact integer, int128)
//     Q    = sum q(t)                           (exact, associative)
//     result = round-half-even-to-fp64(Q) * 2^E_lo
//   The result depends only on the multiset of terms, so any parallel
//   reduction order on the GPU reproduces the oracle bit for bit.
#pragma once
#include <stdint.h>

namespace lap {

typedef __int128 i128;
typedef unsigned __int128 u128;

// SplitMix64 output function (O-S11); bijective on 64-bit words.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t salt_of(uint64_t seed, uint64_t k) {
    return mix64(seed ^ (k * 0x9E3779B97F4A7C15ULL));
}
// uniform [0,1): top 53 bits
__host__ __device__ __forceinline__ double unit_from(uint64_t u) {
    return (double)(u >> 11) * 0x1.0p-53;
}

__host__ __device__ __forceinline__ double __longlong_as_double_hd(long long b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(b);
#else
    double d;
    __builtin_memcpy(&d, &b, sizeof d);
    return d;
#endif
}

__host__ __device__ __forceinline__ int bitlen_u64(uint64_t k) {
#ifdef __CUDA_ARCH__
    return 64 - __clzll((long long)k);
#else
    return k ? 64 - __builtin_clzll(k) : 0;
#endif
}

// E_lo of an instance
__host__ __device__ __forceinline__ int canon_elo(int e_max, int64_t K) {
    return e_max + bitlen_u64((uint64_t)K) - 125;
}

// q(t) = RNE(t * 2^-E_lo), computed in fp64 without bit surgery: the power-of-
// two scaling s = t * 2^-E_lo is exact (|s| < 2^126, and s is normal for any
// finite t because E_lo is far below the exponent of the smallest term that
// matters), rint() is round-half-even, and once |s| >= 2^53 s is already an
// integer that splits exactly into hi * 2^64 + lo.  Same value as the integer
// reference canon_q_bits below (and the oracle's), ~10 instructions instead of
// ~200 (the int128 shift chain made the test-vector sweeps compute-bound).
// 2^-elo when it is a normal double (every realistic instance), else 0: the
// kernels then scale by ONE multiplication -- the correctly rounded product
// t * 2^-elo is exactly scalbn(t, -elo) -- instead of scalbn's special-case
// sequence (the scale is loop-invariant, so it is hoisted out of the loops)
__host__ __device__ __forceinline__ double canon_scale(int elo) {
    return (-elo >= -1022 && -elo <= 1023) ? __longlong_as_double_hd((long long)(1023 - elo) << 52) : 0.0;
}
__device__ __forceinline__ i128 canon_q_s(double t, double s2, int elo) {
    const double sc = s2 != 0.0 ? t * s2 : scalbn(t, -elo);
    if (fabs(sc) < 9007199254740992.0) return (i128)__double2ll_rn(sc);  // |s| < 2^53: RNE to an integer
    const double hi = floor(sc * 0x1p-64);
    const double lo = sc - hi * 0x1p64;                                   // exact, in [0, 2^64)
    return (i128)__double2ll_rz(hi) * ((i128)1 << 64) + (i128)__double2ull_rz(lo);
}
__device__ __forceinline__ i128 canon_q(double t, int elo) { return canon_q_s(t, canon_scale(elo), elo); }

// integer reference of canon_q (bit decomposition); kept for the self-check
__device__ __forceinline__ i128 canon_q_bits(double t, int elo) {
    uint64_t bits = (uint64_t)__double_as_longlong(t);
    uint64_t mag = bits & 0x7FFFFFFFFFFFFFFFULL;
    if (mag == 0) return 0;
    int bexp = (int)(mag >> 52);
    uint64_t man = mag & 0x000FFFFFFFFFFFFFULL;
    int e2;
    if (bexp) {
        man |= 0x0010000000000000ULL;
        e2 = bexp - 1075;
    } else {
        e2 = -1074;
    }
    int sh = e2 - elo;
    u128 q;
    if (sh >= 0) {
        q = ((u128)man) << sh;
    } else {
        int r = -sh;
        if (r > 53) {
            q = 0;
        } else {
            uint64_t keep = man >> r;
            uint64_t rest = man - (keep << r);
            uint64_t half = 1ULL << (r - 1);
            keep += (rest > half) | ((rest == half) & (keep & 1));
            q = keep;
        }
    }
    i128 v = (i128)q;
    return (bits >> 63) ? -v : v;
}

// RNE(Q) * 2^E_lo as fp64
__device__ __forceinline__ double canon_result(i128 Q, int elo) {
    if (Q == 0) return 0.0;
    bool neg = Q < 0;
    u128 a = neg ? (u128)(-(Q + 1)) + 1 : (u128)Q;
    uint64_t hi = (uint64_t)(a >> 64), lo = (uint64_t)a;
    int p = hi ? 127 - __clzll((long long)hi) : 63 - __clzll((long long)lo);
    uint64_t m;
    int e = 0;
    if (p <= 52) {
        m = lo;
    } else {
        int s = p - 52;
        u128 keep = a >> s;
        u128 rest = a - (keep << s);
        u128 half = ((u128)1) << (s - 1);
        if (rest > half || (rest == half && (keep & 1))) keep += 1;
        if (keep >> 53) {
            keep >>= 1;
            s += 1;
        }
        m = (uint64_t)keep;
        e = s;
    }
    double r = scalbn((double)m, e + elo);
    return neg ? -r : r;
}

__device__ __forceinline__ i128 shfl_xor_i128(i128 v, int mask) {
    uint64_t lo = (uint64_t)v, hi = (uint64_t)((u128)v >> 64);
    lo = __shfl_xor_sync(0xffffffffu, lo, mask);
    hi = __shfl_xor_sync(0xffffffffu, hi, mask);
    return (i128)(((u128)hi << 64) | (u128)lo);
}

__device__ __forceinline__ i128 warp_sum_i128(i128 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += shfl_xor_i128(v, o);
    return v;
}

// exponent bound helper: ilogb of a positive finite value (0 -> very small)
__host__ __device__ __forceinline__ int ilogb_pos(double x) {
    if (!(x > 0.0)) return -2000;
#ifdef __CUDA_ARCH__
    return ilogb(x);
#else
    return ilogb(x);
#endif
}

struct I128 {
    unsigned long long lo;
    long long hi;
};
__host__ __device__ __forceinline__ I128 to_I128(i128 v) {
    I128 r;
    r.lo = (unsigned long long)(u128)v;
    r.hi = (long long)(((u128)v) >> 64);
    return r;
}
__host__ __device__ __forceinline__ i128 from_I128(I128 v) {
    return (i128)((((u128)(unsigned long long)v.hi) << 64) | (u128)v.lo);
}
struct I128Add {
    __host__ __device__ __forceinline__ I128 operator()(const I128 &a, const I128 &b) const {
        return to_I128(from_I128(a) + from_I128(b));
    }
};

}  // namespace lap
