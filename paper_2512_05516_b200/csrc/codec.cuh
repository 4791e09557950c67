// Lane codec for the B200 conversion engine.
//
// Storage formats follow the reference's fpcodec (proj/src/fpcodec.cpp:28-155):
// a float lane of total width T is the enclosing IEEE format (binary64 for
// T>=33, binary32 for 17..32, binary16 for 7..16) rounded once with
// round-to-nearest-even, then mantissa-truncated toward zero with a NaN guard.
// bf16 is the new 16-bit mode: narrow_to_ieee(x, 8, 7) (fpcodec.cpp:39-90).
//
// On the device the rounding is the hardware's packed/scalar cvt.rn (F2F,
// F2FP.PACK_AB), which is IEEE RNE with gradual underflow; the only
// disagreement with the reference is NaN (hardware returns a canonical NaN,
// the reference keeps the top payload bits), repaired by a select.  All
// arithmetic is exact except the single RNE, so gather/scatter are bit-exact
// against the reference.
#pragma once
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#define SF_HD __host__ __device__ __forceinline__
#else
#define SF_HD inline
#endif

namespace sfb {

// Base IEEE formats a lane can live in once unpacked.
enum BaseKind : uint8_t { B_F16 = 0, B_BF16 = 1, B_F32 = 2, B_F64 = 3, B_INT = 4 };

struct LaneFmt {
    uint8_t base;   // BaseKind
    uint8_t width;  // stored width in bits (T for compressed lanes, base width when native)
    uint8_t mbits;  // kept mantissa bits (<= base mantissa)
    uint8_t pad;
};

SF_HD int base_width(int base) { return base == B_F64 || base == B_INT ? 64 : base == B_F32 ? 32 : 16; }
SF_HD int base_ebits(int base) { return base == B_F64 ? 11 : base == B_F32 || base == B_BF16 ? 8 : 5; }
SF_HD int base_mbits(int base) { return base == B_F64 ? 52 : base == B_F32 ? 23 : base == B_BF16 ? 7 : 10; }
SF_HD uint64_t lomask(int b) { return b >= 64 ? ~0ull : ((1ull << b) - 1); }

// fpcodec.cpp:28-37: total width -> enclosing base.
SF_HD int base_for_total(int t) { return t >= 33 ? B_F64 : t >= 17 ? B_F32 : B_F16; }

SF_HD LaneFmt fmt_compressed(int t) {  // T-bit stored lane
    LaneFmt f;
    f.base = (uint8_t)base_for_total(t);
    f.width = (uint8_t)t;
    f.mbits = (uint8_t)(t - 1 - base_ebits(f.base));
    f.pad = 0;
    return f;
}
SF_HD LaneFmt fmt_native(int t) {  // T-bit value expanded to its base width
    LaneFmt f = fmt_compressed(t);
    f.width = (uint8_t)base_width(f.base);
    return f;
}
SF_HD LaneFmt fmt_bf16() { LaneFmt f; f.base = B_BF16; f.width = 16; f.mbits = 7; f.pad = 0; return f; }
SF_HD LaneFmt fmt_int() { LaneFmt f; f.base = B_INT; f.width = 64; f.mbits = 0; f.pad = 0; return f; }
SF_HD bool fmt_eq(LaneFmt a, LaneFmt b) { return a.base == b.base && a.width == b.width && a.mbits == b.mbits; }
SF_HD bool fmt_is_ieee(LaneFmt f) { return f.base != B_INT && f.width == base_width(f.base) && f.mbits == base_mbits(f.base); }

// expand_to_base_bits (fpcodec.cpp:119-124): compressed lane -> base bits.
SF_HD uint64_t expand_bits(uint64_t b, LaneFmt f) {
    if (f.base == B_INT || f.width == base_width(f.base)) return b;
    const int bm = base_mbits(f.base), drop = bm - f.mbits;
    return ((b >> f.mbits) << bm) | ((b & lomask(f.mbits)) << drop);
}

// truncate_from_base_bits (fpcodec.cpp:126-135) applied in base space: keep
// the top mbits of the mantissa; a NaN whose kept mantissa would be zero gets
// its top mantissa bit set.  Returns base-width bits.
SF_HD uint64_t trunc_in_base(uint64_t b, int base, int mbits) {
    const int bm = base_mbits(base);
    if (mbits >= bm) return b;
    const int eb = base_ebits(base);
    const uint64_t man = b & lomask(bm);
    const uint64_t kept = man & ~lomask(bm - mbits);
    const bool is_nan = ((b >> bm) & lomask(eb)) == lomask(eb) && man != 0;
    uint64_t out = (b & ~lomask(bm)) | kept;
    if (is_nan && kept == 0) out |= 1ull << (bm - 1);
    return out;
}

// base bits -> compressed storage bits (drop the truncated tail).
SF_HD uint64_t compress_bits(uint64_t base_bits, LaneFmt f) {
    if (f.base == B_INT || f.width == base_width(f.base)) return base_bits;
    const int bm = base_mbits(f.base);
    return ((base_bits >> bm) << f.mbits) | ((base_bits & lomask(bm)) >> (bm - f.mbits));
}

// ---- exact widening of a base-format value to binary64 (widen_from_ieee) ----
SF_HD double bits_to_f64(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
SF_HD uint64_t f64_to_bits(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
SF_HD float bits_to_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
SF_HD uint32_t f32_to_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

SF_HD double nan_widen(uint64_t b, int base) {
    const int bm = base_mbits(base), eb = base_ebits(base);
    const uint64_t s = (b >> (bm + eb)) & 1;
    return bits_to_f64((s << 63) | (0x7ffull << 52) | ((b & lomask(bm)) << (52 - bm)));
}

SF_HD double widen_base(uint64_t b, int base) {
    switch (base) {
        case B_F64: return bits_to_f64(b);
        case B_F32: {
            const uint32_t u = (uint32_t)b;
            if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return nan_widen(b, base);
            return (double)bits_to_f32(u);  // exact
        }
        case B_BF16: {
            const uint32_t u = (uint32_t)(b & 0xffff) << 16;
            if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return nan_widen(b, base);
            return (double)bits_to_f32(u);  // exact
        }
        case B_F16: {
            const uint16_t h = (uint16_t)b;
            if ((h & 0x7c00) == 0x7c00 && (h & 0x3ff)) return nan_widen(b, base);
#ifdef __CUDA_ARCH__
            __half hv;
            memcpy(&hv, &h, 2);
            return (double)__half2float(hv);  // exact
#else
            // host: exact binary16 -> binary64
            const int e = (h >> 10) & 0x1f;
            const uint64_t s = (uint64_t)(h >> 15) << 63;
            uint64_t man = h & 0x3ff;
            if (e == 0x1f) return bits_to_f64(s | (0x7ffull << 52));
            if (e == 0) {
                if (!man) return bits_to_f64(s);
                int lead = 63 - __builtin_clzll(man);
                const int unb = -14 - 10 + lead;
                return bits_to_f64(s | ((uint64_t)(unb + 1023) << 52) | ((man << (52 - lead)) & lomask(52)));
            }
            return bits_to_f64(s | ((uint64_t)(e - 15 + 1023) << 52) | (man << 42));
#endif
        }
    }
    return 0.0;
}

// ---- RNE narrowing of binary64 to a base format (narrow_to_ieee) -------------
// Host version: the integer algorithm, used by the scalar ABI (sf_quantize).
SF_HD uint64_t rne_shift(uint64_t sig, int shift) {
    if (shift <= 0) return sig << -shift;
    if (shift > 64) return 0;
    if (shift == 64) return sig > (1ull << 63) ? 1 : 0;
    const uint64_t q = sig >> shift, r = sig & lomask(shift), half = 1ull << (shift - 1);
    return (r > half || (r == half && (q & 1))) ? q + 1 : q;
}

SF_HD uint64_t narrow_int(double x, int e, int m) {
    const uint64_t src = f64_to_bits(x);
    if (e == 11 && m == 52) return src;
    const uint64_t sign = (src >> 63) << (e + m);
    const int sexp = (int)((src >> 52) & 0x7ff);
    const uint64_t sman = src & lomask(52);
    const int bias = (1 << (e - 1)) - 1, emax = (1 << e) - 1;
    const uint64_t inf = sign | ((uint64_t)emax << m);
    if (sexp == 0x7ff) {
        if (!sman) return inf;
        const uint64_t pay = sman >> (52 - m);
        return inf | (pay ? pay : 1ull << (m - 1));
    }
    uint64_t sig;
    int unb;
    if (sexp == 0) {
        if (!sman) return sign;
#ifdef __CUDA_ARCH__
        const int lead = 63 - __clzll((long long)sman);
#else
        const int lead = 63 - __builtin_clzll(sman);
#endif
        sig = sman << (52 - lead);
        unb = -1022 - (52 - lead);
    } else {
        sig = (1ull << 52) | sman;
        unb = sexp - 1023;
    }
    int texp = unb + bias;
    if (texp >= emax) return inf;
    if (texp >= 1) {
        uint64_t r = rne_shift(sig, 52 - m);
        if (r >> (m + 1)) {
            r >>= 1;
            if (++texp >= emax) return inf;
        }
        return sign | ((uint64_t)texp << m) | (r & lomask(m));
    }
    return sign | rne_shift(sig, (52 - m) + (1 - texp));
}

// NaN repair: what the reference stores for a NaN input (payload = top bits).
SF_HD uint64_t nan_narrow(uint64_t xb, int base) {
    const int bm = base_mbits(base), eb = base_ebits(base);
    const uint64_t sign = (xb >> 63) << (bm + eb);
    uint64_t pay = (xb & lomask(52)) >> (52 - bm);
    if (!pay) pay = 1ull << (bm - 1);
    return sign | (lomask(eb) << bm) | pay;
}

// binary64 -> base bits with RNE.  Device: one hardware cvt.rn + NaN select.
SF_HD uint64_t narrow_base(double x, int base) {
#ifdef __CUDA_ARCH__
    const uint64_t xb = f64_to_bits(x);
    const bool nan = (xb & 0x7fffffffffffffffull) > 0x7ff0000000000000ull;
    uint64_t r;
    switch (base) {
        case B_F64: return xb;
        case B_F32: r = f32_to_bits(__double2float_rn(x)); break;
        case B_BF16: { __nv_bfloat16 b = __double2bfloat16(x); uint16_t u; memcpy(&u, &b, 2); r = u; break; }
        default: { __half h = __double2half(x); uint16_t u; memcpy(&u, &h, 2); r = u; break; }
    }
    return nan ? nan_narrow(xb, base) : r;
#else
    if (base == B_F64) return f64_to_bits(x);
    return narrow_int(x, base_ebits(base), base_mbits(base));
#endif
}

// ---- lane encode / decode ---------------------------------------------------
// decode: stored bits (in format f) -> binary64, exact (decode_bits).
SF_HD double decode_lane(uint64_t bits, LaneFmt f) {
    if (f.base == B_INT) return (double)(int64_t)bits;
    return widen_base(expand_bits(bits, f), f.base);
}

// encode: binary64 -> stored bits in format f (encode_bits; for native lanes
// additionally expand_to_base_bits, BufferView::set sph.cpp:114-126).
SF_HD uint64_t encode_lane(double x, LaneFmt f) {
    if (f.base == B_INT) return (uint64_t)(int64_t)x;
    const uint64_t b = trunc_in_base(narrow_base(x, f.base), f.base, f.mbits);
    return compress_bits(b, f);
}

// bits in format a -> bits in format b (the per-lane rule of the gather).
SF_HD uint64_t convert_lane(uint64_t bits, LaneFmt a, LaneFmt b) {
    if (fmt_eq(a, b)) return bits;
    if (a.base == B_INT || b.base == B_INT) return bits;
    // same base, only a width/truncation change: pure bit transport
    if (a.base == b.base) {
        const uint64_t base = expand_bits(bits, a);
        return compress_bits(trunc_in_base(base, b.base, b.mbits), b);
    }
    return encode_lane(decode_lane(bits, a), b);
}

}  // namespace sfb
