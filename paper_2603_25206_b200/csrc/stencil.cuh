// stencil.cuh — the 7-point gradient + Laplacian emitters and exact statistics shared by the
// windowed (window.cu) and fused (fused.cu) analytics kernels.
// Integer stencils reproduce fields.py:34-80 (derivative: central differences x eps, zero at the
// field edges; Laplacian: 7-point sum x 2 eps, zero on the boundary); outputs are fp32.
#pragma once
#include "common.cuh"

namespace hszg {

__device__ __forceinline__ void acc_add_i128(unsigned long long* limbs, i128 v) {
    const u128 u = (u128)v;
    const unsigned long long l0 = (unsigned long long)(uint32_t)u;
    const unsigned long long l1 = (unsigned long long)(uint32_t)(u >> 32);
    const unsigned long long l2 = (unsigned long long)(uint32_t)(u >> 64);
    const long long l3 = (long long)(int32_t)(uint32_t)(u >> 96);   // signed top limb
    if (l0) atomicAdd(limbs + 0, l0);
    if (l1) atomicAdd(limbs + 1, l1);
    if (l2) atomicAdd(limbs + 2, l2);
    if (l3) atomicAdd(limbs + 3, (unsigned long long)l3);
}

struct WinStats {
    int64_t s1_64;   // per-thread partial: <= 4*W terms of |q| < 2^31
    uint64_t sq;     // fast-path partial of q^2 (|q| < 2^27: four squares < 2^56), folded every <= 32 add4f
    i128 s1, s2;
    int32_t vmin, vmax;
    __device__ __forceinline__ void init() {
        s1_64 = 0;
        sq = 0;
        s1 = 0;
        s2 = 0;
        vmin = INT32_MAX;
        vmax = INT32_MIN;
    }
    __device__ __forceinline__ void add4(int4 q) {
        s1_64 += (int64_t)q.x + q.y + q.z + q.w;
        // four squares < 4 * 2^62 = 2^64: exact in u64, one 128-bit add per four values
        const uint64_t sq4 = (uint64_t)((int64_t)q.x * q.x) + (uint64_t)((int64_t)q.y * q.y) +
                             (uint64_t)((int64_t)q.z * q.z) + (uint64_t)((int64_t)q.w * q.w);
        s2 += (i128)(u128)sq4;
        vmin = min(vmin, min(min(q.x, q.y), min(q.z, q.w)));
        vmax = max(vmax, max(max(q.x, q.y), max(q.z, q.w)));
    }
    // fast-path variant, exact while |q| < 2^27 (FAST_QLIM) — the condition the caller verifies from
    // vmin / vmax (always exact) before trusting the fast pass; call fold() at least every 32 calls
    __device__ __forceinline__ void add4f(int4 q) {
        s1_64 += (int64_t)((q.x + q.y) + (q.z + q.w));
        // chained 64-bit multiply-adds (one IMAD.WIDE each); |q| < 2^27 keeps 128 squares < 2^63
        int64_t t = (int64_t)sq;
        t += (int64_t)q.x * q.x;
        t += (int64_t)q.y * q.y;
        t += (int64_t)q.z * q.z;
        t += (int64_t)q.w * q.w;
        sq = (uint64_t)t;
        vmin = min(vmin, min(min(q.x, q.y), min(q.z, q.w)));
        vmax = max(vmax, max(max(q.x, q.y), max(q.z, q.w)));
    }
    __device__ __forceinline__ void fold() {
        s2 += (i128)(u128)sq;
        sq = 0;
    }
    // warp-reduce, then one lane publishes
    __device__ __forceinline__ void flush(HszgAcc* acc, int64_t count) {
        fold();
        s1 += s1_64;
        for (int d = 16; d > 0; d >>= 1) {
            s1 += shfl_down_i128(s1, d);
            s2 += shfl_down_i128(s2, d);
            vmin = min(vmin, __shfl_down_sync(0xffffffffu, vmin, d));
            vmax = max(vmax, __shfl_down_sync(0xffffffffu, vmax, d));
            count += __shfl_down_sync(0xffffffffu, count, d);
        }
        if ((threadIdx.x & 31) == 0 && count) {
            acc_add_i128(reinterpret_cast<unsigned long long*>(acc->s1_limb), s1);
            acc_add_i128(reinterpret_cast<unsigned long long*>(acc->s2_limb), s2);
            atomicAdd(reinterpret_cast<unsigned long long*>(&acc->count), (unsigned long long)count);
            atomicMin(&acc->vmin, vmin);
            atomicMax(&acc->vmax, vmax);
        }
    }
};

__device__ __forceinline__ float4 sc4(int64_t a, int64_t b, int64_t c, int64_t d, double s) {
    return make_float4(__double2float_rn(__dmul_rn((double)a, s)), __double2float_rn(__dmul_rn((double)b, s)),
                       __double2float_rn(__dmul_rn((double)c, s)), __double2float_rn(__dmul_rn((double)d, s)));
}

__device__ __forceinline__ int4 add4(int4 a, int4 b) {
    return make_int4((int)((uint32_t)a.x + (uint32_t)b.x), (int)((uint32_t)a.y + (uint32_t)b.y),
                     (int)((uint32_t)a.z + (uint32_t)b.z), (int)((uint32_t)a.w + (uint32_t)b.w));
}

__device__ __forceinline__ int4 ld4(const int32_t* p) { return __ldg(reinterpret_cast<const int4*>(p)); }

// Emit gradient (dz, dy, dx) + Laplacian for 4 x-points given the 7-point neighbourhood.
// OM: outputs written (bit 0 dz, 1 dy, 2 dx, 3 Laplacian; OM_ALL, OM_GRAD or OM_LAP) — the API's derivative /
// Laplacian calls skip the other outputs' arithmetic and stores
enum OutMask { OM_GRAD = 7, OM_LAP = 8, OM_ALL = 15 };
template <int OM = OM_ALL>
__device__ __forceinline__ void emit4(float* o0, float* o1, float* o2, float* o3, int64_t o, bool zin, bool yin,
                                      int64_t xi, int64_t n2, int4 zm, int4 c, int4 zp, int4 ym, int4 yp,
                                      int32_t left, int32_t right, double eps, double two_eps) {
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 dz = zero, dy = zero, lp = zero, dx = zero;
    if ((OM & 1) && zin) dz = sc4((int64_t)zp.x - zm.x, (int64_t)zp.y - zm.y, (int64_t)zp.z - zm.z, (int64_t)zp.w - zm.w, eps);
    if ((OM & 2) && yin) dy = sc4((int64_t)yp.x - ym.x, (int64_t)yp.y - ym.y, (int64_t)yp.z - ym.z, (int64_t)yp.w - ym.w, eps);
    if (OM & 4) {
        int64_t d0 = (int64_t)c.y - left, d1 = (int64_t)c.z - c.x, d2 = (int64_t)c.w - c.y, d3 = (int64_t)right - c.z;
        if (xi == 0) d0 = 0;
        if (xi + 3 >= n2 - 1) d3 = 0;
        dx = sc4(d0, d1, d2, d3, eps);
    }
    if ((OM & 8) && zin && yin) {
        int64_t l0 = (int64_t)zm.x + zp.x + ym.x + yp.x + left + c.y - 6ll * c.x;
        int64_t l1 = (int64_t)zm.y + zp.y + ym.y + yp.y + c.x + c.z - 6ll * c.y;
        int64_t l2 = (int64_t)zm.z + zp.z + ym.z + yp.z + c.y + c.w - 6ll * c.z;
        int64_t l3 = (int64_t)zm.w + zp.w + ym.w + yp.w + c.z + right - 6ll * c.w;
        if (xi == 0) l0 = 0;
        if (xi + 3 >= n2 - 1) l3 = 0;
        lp = sc4(l0, l1, l2, l3, two_eps);
    }
    if (OM & 1) __stcs(reinterpret_cast<float4*>(o0 + o), dz);
    if (OM & 2) __stcs(reinterpret_cast<float4*>(o1 + o), dy);
    if (OM & 4) __stcs(reinterpret_cast<float4*>(o2 + o), dx);
    if (OM & 8) __stcs(reinterpret_cast<float4*>(o3 + o), lp);
}

// Fast fp32 emitter (the pipeline default): integer stencils in int32 (I2FP converts on the ALU
// pipe) times the fp32-rounded scale: within 4 * 2^-24 relative of fl32(D*eps) (<< 1e-6).
// Requires |q| < 2^27 over the neighbourhood (the int32 Laplacian cannot overflow); the caller
// checks that afterwards from the exact min/max statistics (every q is some point's centre) and
// re-runs the exact emitter if it was violated (FAST_QLIM; pipeline.py).
constexpr int32_t FAST_QLIM = 1 << 27;
__device__ __forceinline__ float4 sc4f(int32_t a, int32_t b, int32_t c, int32_t d, float s) {
    return make_float4(__int2float_rn(a) * s, __int2float_rn(b) * s, __int2float_rn(c) * s, __int2float_rn(d) * s);
}

__device__ __forceinline__ void emit4f(float* o0, float* o1, float* o2, float* o3, int64_t o, bool zin, bool yin,
                                       int64_t xi, int64_t n2, int4 zm, int4 c, int4 zp, int4 ym, int4 yp,
                                       int32_t left, int32_t right, double, double, float epsf, float two_epsf) {
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 dz = zero, dy = zero, lp = zero;
    if (zin) dz = sc4f(zp.x - zm.x, zp.y - zm.y, zp.z - zm.z, zp.w - zm.w, epsf);
    if (yin) dy = sc4f(yp.x - ym.x, yp.y - ym.y, yp.z - ym.z, yp.w - ym.w, epsf);
    int32_t d0 = c.y - left, d1 = c.z - c.x, d2 = c.w - c.y, d3 = right - c.z;
    if (xi == 0) d0 = 0;
    if (xi + 3 >= n2 - 1) d3 = 0;
    const float4 dx = sc4f(d0, d1, d2, d3, epsf);
    if (zin && yin) {
        int32_t l0 = zm.x + zp.x + ym.x + yp.x + left + c.y - 6 * c.x;
        int32_t l1 = zm.y + zp.y + ym.y + yp.y + c.x + c.z - 6 * c.y;
        int32_t l2 = zm.z + zp.z + ym.z + yp.z + c.y + c.w - 6 * c.z;
        int32_t l3 = zm.w + zp.w + ym.w + yp.w + c.z + right - 6 * c.w;
        if (xi == 0) l0 = 0;
        if (xi + 3 >= n2 - 1) l3 = 0;
        lp = sc4f(l0, l1, l2, l3, two_epsf);
    }
    __stcs(reinterpret_cast<float4*>(o0 + o), dz);
    __stcs(reinterpret_cast<float4*>(o1 + o), dy);
    __stcs(reinterpret_cast<float4*>(o2 + o), dx);
    __stcs(reinterpret_cast<float4*>(o3 + o), lp);
}

// Exact fp32 emitter by table (emitter mode EM_TABLE): the outputs are fl32(fl64(D * eps)) of the integer
// stencil D, bit-identical to emit4, but the fp64 conversion chain (I2F.F64 + DMUL + F2F.F32.F64, slow pipes)
// runs only for |D| >= XT_R: T[D] = fl32(fl64(D * eps)) for |D| < XT_R sits in shared memory, filled by the
// CTA at start.  The Laplacian uses 2 * T[L]: fl64(L * 2 eps) = 2 fl64(L * eps) and fl32(2 v) = 2 fl32(v)
// while every result is a normal float (host guard: eps in [2^-125, 2^90]).  Integer stencils in int32 as
// in emit4f, so the caller checks |q| < FAST_QLIM afterwards (exact min / max) and re-runs emit4 otherwise.
enum EmitMode { EM_FAST = 0, EM_EXACT = 1, EM_TABLE = 2 };
constexpr int XT_R = 2048;                       // table half range: D in [-XT_R, XT_R)
constexpr int XT_BYTES = 2 * XT_R * 4;
__device__ __forceinline__ void xtable_fill(float* T, double eps, int tid, int nthreads) {
    for (int i = tid; i < 2 * XT_R; i += nthreads) T[i] = __double2float_rn(__dmul_rn((double)(i - XT_R), eps));
}
__device__ __forceinline__ bool xin(int32_t d) { return (uint32_t)(d + XT_R) < (uint32_t)(2 * XT_R); }
__device__ __forceinline__ float4 xt4(int4 d, const float* Tc) {      // Tc = T + XT_R (centre)
    return make_float4(Tc[d.x], Tc[d.y], Tc[d.z], Tc[d.w]);
}
__device__ __forceinline__ float4 xs4(int4 d, double eps) {             // the conversion chain (rare)
    return make_float4(__double2float_rn(__dmul_rn((double)d.x, eps)), __double2float_rn(__dmul_rn((double)d.y, eps)),
                       __double2float_rn(__dmul_rn((double)d.z, eps)), __double2float_rn(__dmul_rn((double)d.w, eps)));
}

// The 16 integer stencil values are formed first; the warp takes the table path unless one of its lanes has
// a value outside the table (then the whole warp runs the conversion chain for this row: uniform branch,
// so the common path never issues fp64 work under predication).
template <int OM, typename OffT>
__device__ __forceinline__ void emit4x(float* o0, float* o1, float* o2, float* o3, OffT o, bool zin, bool yin,
                                       int64_t xi, int64_t n2, int4 zm, int4 c, int4 zp, int4 ym, int4 yp,
                                       int32_t left, int32_t right, double eps, const float* Tc) {
    const int4 z4 = make_int4(0, 0, 0, 0);
    int4 dz = z4, dy = z4, dx = z4, lp = z4;
    if ((OM & 1) && zin) dz = make_int4(zp.x - zm.x, zp.y - zm.y, zp.z - zm.z, zp.w - zm.w);
    if ((OM & 2) && yin) dy = make_int4(yp.x - ym.x, yp.y - ym.y, yp.z - ym.z, yp.w - ym.w);
    if (OM & 4) {
        dx = make_int4(c.y - left, c.z - c.x, c.w - c.y, right - c.z);
        if (xi == 0) dx.x = 0;
        if (xi + 3 >= n2 - 1) dx.w = 0;
    }
    if ((OM & 8) && zin && yin) {
        lp.x = zm.x + zp.x + ym.x + yp.x + left + c.y - 6 * c.x;
        lp.y = zm.y + zp.y + ym.y + yp.y + c.x + c.z - 6 * c.y;
        lp.z = zm.z + zp.z + ym.z + yp.z + c.y + c.w - 6 * c.z;
        lp.w = zm.w + zp.w + ym.w + yp.w + c.z + right - 6 * c.w;
        if (xi == 0) lp.x = 0;
        if (xi + 3 >= n2 - 1) lp.w = 0;
    }
    // range of the written values by min / max (fewer instructions than one compare each)
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    auto rng = [&](int4 v) {
        lo = min(lo, min(min(v.x, v.y), min(v.z, v.w)));
        hi = max(hi, max(max(v.x, v.y), max(v.z, v.w)));
    };
    if (OM & 1) rng(dz);
    if (OM & 2) rng(dy);
    if (OM & 4) rng(dx);
    if (OM & 8) rng(lp);
    const bool in = lo >= -XT_R && hi < XT_R;
    float4 fz, fy, fx, fl;
    if (__all_sync(__activemask(), in)) {     // callers may run this under a per-lane edge predicate
        if (OM & 1) fz = xt4(dz, Tc);
        if (OM & 2) fy = xt4(dy, Tc);
        if (OM & 4) fx = xt4(dx, Tc);
        if (OM & 8) fl = xt4(lp, Tc);
    } else {
        if (OM & 1) fz = xs4(dz, eps);
        if (OM & 2) fy = xs4(dy, eps);
        if (OM & 4) fx = xs4(dx, eps);
        if (OM & 8) fl = xs4(lp, eps);
    }
    if (OM & 1) __stcs(reinterpret_cast<float4*>(o0 + o), fz);
    if (OM & 2) __stcs(reinterpret_cast<float4*>(o1 + o), fy);
    if (OM & 4) __stcs(reinterpret_cast<float4*>(o2 + o), fx);
    if (OM & 8) __stcs(reinterpret_cast<float4*>(o3 + o), make_float4(2.0f * fl.x, 2.0f * fl.y, 2.0f * fl.z, 2.0f * fl.w));
}

__device__ __forceinline__ int4 add4u(int4 a, uint32_t o) {
    return make_int4((int)((uint32_t)a.x + o), (int)((uint32_t)a.y + o), (int)((uint32_t)a.z + o),
                     (int)((uint32_t)a.w + o));
}

}  // namespace hszg
