// swar.cuh -- byte-SIMD helpers for the P-HGRMS stencil on sm_100a.
//
// Four pixels travel in one 32-bit word (byte j = column c+j).  The
// similarity test of the reference, similar(a,b,alpha) = |a-b| < alpha
// (include/phgrms/denoise.hpp:88), is evaluated for four pixel pairs at once:
//
//   d   = VABSDIFF4(a, b)                       (native SASS VABSDIFF4.U8)
//   t   = (d & 0x7f7f7f7f) + k7,  k = 256-alpha (per byte, k7 = k & 0x7f)
//   dis = carry out of d+k   = MAJ(d7, k7, t7) (bit 7 of each byte)
//
// d+k >= 256  <=>  d >= alpha, so `dis` is exactly !similar.  For
// alpha <= 128 the top bit of k is 1 and MAJ reduces to d|t (one LOP3 with
// the validity mask folded in); for alpha > 128 it is d&t.
#pragma once
#include <cstdint>

namespace phg {

constexpr uint32_t kHi = 0x80808080u;
constexpr uint32_t kLo7 = 0x7f7f7f7fu;

// 0x80 in every byte lane where |a-b| < alpha and `valid` has its 0x80 bit.
template <bool ALPHA_LE128>
__device__ __forceinline__ uint32_t sim_bits(uint32_t a, uint32_t b, uint32_t k7,
                                             uint32_t valid) {
    const uint32_t d = __vabsdiffu4(a, b);
    const uint32_t t = (d & kLo7) + k7;
    const uint32_t dis = ALPHA_LE128 ? (d | t) : (d & t);
    return valid & ~dis;
}

// Per-byte c < thr for small counts (c <= 127, thr in [1,127]):
// c + (128-thr) stays inside the byte, its bit 7 is clear iff c < thr.
__device__ __forceinline__ uint32_t lt_bits(uint32_t c, uint32_t k_thr) {
    return ~(c + k_thr) & kHi;
}

__device__ __forceinline__ uint32_t rep4(uint32_t b) { return b * 0x01010101u; }

// 0xff in every byte whose bit 7 is set (PRMT sign-replicate mode; note that
// the __byte_perm intrinsic masks the selector's replicate bit away).
__device__ __forceinline__ uint32_t msb_to_bytes(uint32_t x) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xba98;" : "=r"(r) : "r"(x));
    return r;
}

// round-half-away-from-zero of sqrt(S/f), exactly as the reference's
// llround(sqrt(double(S)/f)) (denoise.hpp:163-169): u is the largest
// integer with u - 1/2 <= sqrt(S/f), i.e. (2u-1)^2 * f <= 4S (u >= 1), or 0.
// The fp32 estimate is corrected with exact integer tests, so the result is
// exact by construction for every reachable (S, f).
__device__ __forceinline__ uint32_t rms_round(uint64_t S, uint32_t f) {
    const float est = sqrtf(static_cast<float>(S) / static_cast<float>(f));
    int64_t u = static_cast<int64_t>(est + 0.5f);
    const uint64_t S4 = S * 4u;
    while (u >= 1 && static_cast<uint64_t>((2 * u - 1) * (2 * u - 1)) * f > S4) --u;
    while (static_cast<uint64_t>((2 * u + 1) * (2 * u + 1)) * f <= S4) ++u;
    return u > 255 ? 255u : static_cast<uint32_t>(u);
}

}  // namespace phg
