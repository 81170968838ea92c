// trigbf_b200.cu -- B200 (sm_100a) constant-time trigonometric bilateral filter.
//
// Reference semantics: /root/reference/pkg/src/trigbf/engines.py:228-306
// (bilateral_trig) with spatial.py:163-182 (separable recursive Gaussian /
// box smoother) and _core.pyx:28-96 (the two compiled loops).
//
// Pipeline per term batch (see DESIGN.md for the derivation and roofline):
//
//   k_transpose    f -> fT (x-major, for pass 2) and fY (tile-major, for
//                  pass 1), fused with the input range check.
//   k_pass1_gauss  one warp = 32 adjacent columns x one term.  The four
//                  auxiliary planes of the term (cos, sin, f*cos, f*sin of
//                  nu*f) are generated in registers from f and run through
//                  the forward/backward biquad cascade along y.  The
//                  causal->anticausal dependency is broken with per-32-row
//                  checkpoints of the forward state (phase A) and a segment-
//                  wise recompute into shared memory (phase B).  The segment
//                  tile is then read transposed from shared memory and the
//                  zero-state forward recursion along x is run over the 32
//                  columns of the tile ("tile-local forward"), which is what is
//                  written to HBM (one fp32 round trip of the 4 planes).
//   k_chain        per (row, term): chains the 4-state carries of the tiles
//                  along x (s' = M s + L), handles the mirrored x-extension
//                  (the right one in closed form), and produces the backward
//                  start state.
//   k_pass2_gr     one warp = 32 rows x G2 terms, 4 warps (term groups) per
//                  block, tiles right to left: exact forward output =
//                  tile-local + H[m] . carry, then the backward cascade,
//                  demodulation and num/den accumulation in registers; the
//                  block sums its 4 groups in shared memory (fixed order).
//   k_reduce       folds the per-block partial num/den, transposes back to
//                  row-major and applies the guarded ratio (engines.py:109-117).
//
// No tensor cores: the path is a set of first/second-order linear
// recurrences, bounded by HBM bandwidth and the FP32 pipe.

#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <queue>
#include <tuple>
#include <cmath>
#include <string>
#include <vector>

#ifndef TBF_PHASOR_SFU
#define TBF_PHASOR_SFU 2  // 1: SFU after an explicit 2*pi reduction; 0: FMA-pipe polynomial (see sincos_fma)
#endif

#include "trigbf_b200.h"

#define TBF_ABI_VERSION 2

namespace {

#ifndef TBF_P1_ASTORE
#define TBF_P1_ASTORE 0  // 1: phase A also writes every segment tile (the round-1/2 code)
#endif
constexpr int TILE = 32;          // segment length along y == tile width along x == warp size
constexpr int P1_WARPS = 4;       // warps per pass-1 block (each a different term group)
constexpr int P2_THREADS = 128;   // rows per pass-2 block
constexpr int FL_RB = 32;         // row-block height of the x-major tiling: one pass-2 warp's rows,
                                  // so a warp streams 512 contiguous bytes per x-step and its
                                  // consecutive x-steps are adjacent

// x-major per-pixel planes read by pass 2 (fT, partial num/den, and F_loc per
// term) are row-block tiled: [b][row block of 32][x][32 rows], so a pass-2
// warp streams its rows contiguously as x advances.
__host__ __device__ __forceinline__ size_t xm_index(int b, int x, int i, int W, int H) {
    const int nrb = (H + FL_RB - 1) / FL_RB;
    return (((size_t)b * nrb + i / FL_RB) * W + x) * FL_RB + (i % FL_RB);
}
// Tile-major copy of f read by pass 1: [b][row tile][column tile][32][32],
// so the 32 rows of a warp's 32 columns are 4 KB contiguous (row loads are
// coalesced 128 B with immediate offsets from one base address).
__host__ __device__ __forceinline__ size_t ty_index(int b, int x, int i, int W, int H) {
    const int nys = (H + 31) / 32, ntx = (W + 31) / 32;
    return ((((size_t)b * nys + i / 32) * ntx + x / 32) * 32 + (i % 32)) * 32 + (x % 32);
}
__host__ __device__ __forceinline__ size_t ty_plane(int B, int W, int H) {
    return (size_t)B * ((H + 31) / 32) * 32 * ((W + 31) / 32) * 32;
}
__host__ __device__ __forceinline__ size_t xm_plane(int B, int W, int H) {
    return (size_t)B * ((H + FL_RB - 1) / FL_RB) * FL_RB * W;
}
constexpr int TBF_MAX_YCH = 16;      // most y-chunks per pass-1 column
constexpr int P1_MAX_LAUNCHES = 64;  // pass-1 launches per batch (host strips), one dispatch ticket each
constexpr int P1_BLOCKS_PER_SM = 3;  // smem-limited residency of pass-1 blocks (4 warps, 67.6 KB)
constexpr int BUF_LD = TILE + 1;  // padded leading dimension of the smem tile
constexpr int STRIPE = P1_WARPS * TILE;  // columns per pass-1 block (x carries are chained per stripe)

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int check_cuda(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TBF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return TBF_OK;
}

// Optional per-kernel timing: CUDA events recorded on the launch stream around
// every launch (tbf_profile_enable / tbf_profile_collect).
enum KernelKind {
    KK_TRANSPOSE = 0, KK_RANGE, KK_PASS1, KK_CHAIN, KK_PASS2, KK_REDUCE, KK_FINALIZE, KK_H2D, KK_D2H,
    KK_COUNT
};
const char* const kKernelNames[KK_COUNT] = {"transpose", "range_check", "pass1", "edge",
                                            "pass2", "reduce", "finalize", "h2d", "d2h"};

struct ProfRec {
    int kind;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_ev_pool;

cudaEvent_t ev_get() {
    if (!g_ev_pool.empty()) {
        cudaEvent_t e = g_ev_pool.back();
        g_ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct Prof {
    int kind;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    Prof(int k, cudaStream_t s) : kind(k), st(s) {
        std::lock_guard<std::mutex> g(g_prof_mu);
        if (g_prof_on) {
            a = ev_get();
            cudaEventRecord(a, st);
        }
    }
    ~Prof() {
        if (!a) return;
        std::lock_guard<std::mutex> g(g_prof_mu);
        cudaEvent_t b = ev_get();
        cudaEventRecord(b, st);
        g_prof.push_back({kind, a, b});
    }
};

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------

// Cascade of the two pole-pair sections in "pure" form: the section gains
// g1, g2 are not applied per sample (v = u + a1 v1 + a2 v2; y = v + b1 y1 +
// b2 y2: 4 FMA per sample instead of 6).  Each pure sweep therefore scales
// its output by 1/g (g = g1*g2); the host folds the scale back in (pass-1
// epilogue multiplies by gg = g^2, pass-2 weights carry g^2).
struct Casc {
    float a1, a2, b1, b2;
    float ig1;  // 1/g1  (steady state of section 1 for unit input)
    float ig;   // 1/g   (steady state of the cascade for unit input)
    float gg;   // g^2   (undoes the two y sweeps)
};

// Whole-sample reflection for indices within one reflection of the line
// (|extension| <= n-1), identical to _mirror (_core.pyx:14-25) there.
__device__ __forceinline__ int mirror1(int i, int n) {
    i = i < 0 ? -i : i;
    return i >= n ? 2 * (n - 1) - i : i;
}

// General whole-sample reflection (period 2(n-1)), _core.pyx:14-25.
__device__ __forceinline__ long long mirror_any(long long i, long long n) {
    if (n == 1) return 0;
    long long period = 2 * (n - 1);
    i %= period;
    if (i < 0) i += period;
    return i >= n ? period - i : i;
}



// F_loc is written once (pass 1) and read once (pass 2), far apart: with
// TBF_CACHE_HINTS its stores and loads are streaming (evict-first), so the
// 16 B/pixel-term stream does not evict the L2-resident f tile copy,
// checkpoints and carries.
#ifndef TBF_CACHE_HINTS
#define TBF_CACHE_HINTS 1
#endif
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
#if TBF_CACHE_HINTS
    __stcs(p, v);
#else
    *p = v;
#endif
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
#if TBF_CACHE_HINTS
    return __ldcs(p);
#else
    return *p;
#endif
}

// Read-only global load kept in program order relative to the surrounding
// shared-memory stores (volatile + memory clobber): pins prefetches where the
// source puts them instead of letting them sink next to their use.
__device__ __forceinline__ float ldg_pinned(const float* p) {
    float v;
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}

// Flag hand-off between blocks (the pass-1 x chain): release store by the
// producer after its data.
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Consumer side without acquire semantics (an acquire costs an L1
// invalidation, CCTL.IVALL, per hand-off and the block's warps share f rows
// in L1): the flag is polled with strong relaxed loads and the data read with
// strong loads that are only issued once the poll loop has seen the flag, so
// both are served by L2, where the producer's release made the data visible
// before the flag.
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ float4 ld_relaxed4(const float4* p) {
    float4 v;
    asm volatile("ld.relaxed.gpu.global.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

// Thread-block clusters (the pass-1 x hand-off between the stripes of a
// cluster through distributed shared memory and mbarriers).
__device__ __forceinline__ unsigned cluster_ctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t map_cluster(uint32_t saddr, unsigned rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_init_cta(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cbar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cbar) : "memory");
}
// wait for the phase with the given parity to complete (trap after ~10 s)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
    const uint32_t a = smem_addr(bar);
    unsigned spins = 0;
    for (;;) {
        uint32_t done;
        asm volatile(
            "{\n.reg .pred P;\n"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P;\n}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
        if (done) return;
        if (++spins == (1u << 26)) __trap();
    }
}
__device__ __forceinline__ void st_cluster4(uint32_t caddr, float4 v) {
    asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(caddr), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ unsigned ld_cluster_u32(uint32_t caddr) {
    unsigned v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(caddr) : "memory");
    return v;
}

// Named barriers between pairs of warps (the pass-1 x hand-off inside a
// block): arrive does not wait; sync waits for `count` threads in total.
// Barrier ids are immediates (ptxas then reserves ids 0..7 only, not all 16):
// FULL 1 + w and EMPTY 5 + w for the links w -> w+1, w = 0..2.
#define TBF_BAR_CASE(op, n) \
    case n: asm volatile(op " " #n ", 64;" ::: "memory"); break;
__device__ __forceinline__ void named_bar_sync(int id, int /*count = 64*/) {
    switch (id) {
        TBF_BAR_CASE("bar.sync", 1)
        TBF_BAR_CASE("bar.sync", 2)
        TBF_BAR_CASE("bar.sync", 3)
        TBF_BAR_CASE("bar.sync", 4)
        TBF_BAR_CASE("bar.sync", 5)
        TBF_BAR_CASE("bar.sync", 6)
        TBF_BAR_CASE("bar.sync", 7)
        default: __trap();
    }
}
__device__ __forceinline__ void named_bar_arrive(int id, int /*count = 64*/) {
    switch (id) {
        TBF_BAR_CASE("bar.arrive", 1)
        TBF_BAR_CASE("bar.arrive", 2)
        TBF_BAR_CASE("bar.arrive", 3)
        TBF_BAR_CASE("bar.arrive", 4)
        TBF_BAR_CASE("bar.arrive", 5)
        TBF_BAR_CASE("bar.arrive", 6)
        TBF_BAR_CASE("bar.arrive", 7)
        default: __trap();
    }
}
#undef TBF_BAR_CASE
static_assert(P1_WARPS == 4, "pass-1 hand-off barrier ids 1..7 assume 4 warps per block");

// One pure cascade step (state v1,v2 | y1,y2); output scaled by 1/g.
__device__ __forceinline__ float cstep(float u, float& v1, float& v2, float& y1, float& y2,
                                       const Casc& k) {
    float v = fmaf(k.a1, v1, fmaf(k.a2, v2, u));
    v2 = v1;
    v1 = v;
    float y = fmaf(k.b1, y1, fmaf(k.b2, y2, v));
    y2 = y1;
    y1 = y;
    return y;
}

// Steady state of the pure cascade for a constant input u (replicate
// start-up of _core.pyx:75-78 / :85-87).
__device__ __forceinline__ void csteady(float u, float& v1, float& v2, float& y1, float& y2,
                                        const Casc& k) {
    v1 = v2 = u * k.ig1;
    y1 = y2 = u * k.ig;
}

// Phase nu * f with nu split hi/lo (TBF_PHASE_HILO=1, default: correctly
// rounded) or nu_hi * f alone (0).
#ifndef TBF_PHASE_HILO
#define TBF_PHASE_HILO 1
#endif
__device__ __forceinline__ float phase(float nu_hi, float nu_lo, float f) {
#if TBF_PHASE_HILO
    return fmaf(nu_hi, f, nu_lo * f);
#else
    (void)nu_lo;
    return nu_hi * f;
#endif
}

// sin and cos of x for |x| < ~1e5.  TBF_PHASOR_SFU=2 (default): SFU directly;
// 1: SFU after an explicit 2*pi reduction; 0: FMA pipe only (no SFU, no
// slow-path branch): Cody-Waite reduction by pi/2 in three parts (exact products inside
// the FMAs), then the Cephes minimax polynomials on [-pi/4, pi/4] (about 1 ulp).
// Arguments here are nu*f <= ~420 rad.
__device__ __forceinline__ void sincos_fma(float x, float* sp, float* cp) {
#if TBF_PHASOR_SFU == 2
    // default: the SFU directly (FMUL.RZ by 1/(2 pi), MUFU.SIN/COS take the
    // fraction of the turn count themselves).  Phase error ~1 ulp of
    // x/(2 pi) (~1e-5 rad at config 2's largest phase, ~5e-5 at config 3's)
    // instead of ~1 ulp of x; 5 instructions instead of 9, measured 2-3%
    // faster end to end with parity unchanged
    __sincosf(x, sp, cp);
#elif TBF_PHASOR_SFU
    // Cody-Waite reduction by 2*pi in two parts (q*6.28125 exact for
    // q < 2^15), then the SFU (MUFU.SIN/COS, abs error ~2^-21 on [-pi, pi]).
    // 9 instructions instead of ~24 for the polynomial; measured +10% end to
    // end on configs 2/3/5 with unchanged parity
    const float t = fmaf(x, 0.159154943091895336f, 12582912.0f);
    const float q = t - 12582912.0f;
    float r = fmaf(q, -6.28125f, x);
    r = fmaf(q, -1.9353071795864769e-3f, r);
    __sincosf(r, sp, cp);
#else
    // q = nearest integer to x*2/pi via the 1.5*2^23 magic constant (its low
    // mantissa bits hold q), no F2I / FRND
    const float t = fmaf(x, 0.636619772367581343f, 12582912.0f);
    const float q = t - 12582912.0f;
    const int qi = __float_as_int(t);
    float r = fmaf(q, -1.5703125f, x);
    r = fmaf(q, -4.837512969970703125e-4f, r);
    r = fmaf(q, -7.54978995489188216e-8f, r);
    const float r2 = r * r;
    float ps = fmaf(r2, -1.9515295891e-4f, 8.3321608736e-3f);
    ps = fmaf(r2, ps, -1.6666654611e-1f);
    ps = fmaf(r2 * r, ps, r);
    float pc = fmaf(r2, 2.443315711809948e-5f, -1.388731625493765e-3f);
    pc = fmaf(r2, pc, 4.166664568298827e-2f);
    pc = fmaf(r2, pc, -0.5f);
    pc = fmaf(r2, pc, 1.0f);
    const bool swap = qi & 1;
    float sv = swap ? pc : ps;
    float cv = swap ? ps : pc;
    sv = __int_as_float(__float_as_int(sv) ^ ((qi & 2) << 30));
    cv = __int_as_float(__float_as_int(cv) ^ (((qi + 1) & 2) << 30));
    *sp = sv;
    *cp = cv;
#endif
}

// Phasors of G consecutive terms at one sample (engines.py:272-286).  Terms
// are grouped in anchor blocks of R: the first term of a block takes an
// accurate sincos of nu*f (nu split hi/lo so the phase is correctly rounded),
// the others follow by complex rotation with (cos, sin)(dnu*f).  Pass 1 and
// pass 2 use the same rule, so modulation and demodulation see bit-identical
// phasors.
template <int G, int R>
__device__ __forceinline__ void phasors(float fv, const float (&nu_hi)[G], const float (&nu_lo)[G],
                                        float dnu, float (&cc)[G], float (&sn)[G]) {
    float ss = 0.f, sc = 1.f;
    if (R > 1) sincos_fma(dnu * fv, &ss, &sc);
    float c = 1.f, s = 0.f;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        if (g % R == 0) {
            sincos_fma(phase(nu_hi[g], nu_lo[g], fv), &s, &c);
        } else {
            float cn = fmaf(c, sc, -s * ss);
            float snn = fmaf(s, sc, c * ss);
            c = cn;
            s = snn;
        }
        cc[g] = c;
        sn[g] = s;
    }
}

// Auxiliary planes u[4g+0..3] = cos, sin, f*cos, f*sin (engines.py:287).
template <int G, int R>
__device__ __forceinline__ void modulate(float fv, const float (&nu_hi)[G], const float (&nu_lo)[G],
                                         float dnu, float (&u)[4 * G]) {
    float cc[G], sn[G];
    phasors<G, R>(fv, nu_hi, nu_lo, dnu, cc, sn);
#pragma unroll
    for (int g = 0; g < G; ++g) {
        u[4 * g + 0] = cc[g];
        u[4 * g + 1] = sn[g];
        u[4 * g + 2] = fv * cc[g];
        u[4 * g + 3] = fv * sn[g];
    }
}


// ---------------------------------------------------------------------------
// Block helpers: NB consecutive samples of one line.  Phasors of all NB
// samples are computed first (independent -> overlapped by the scheduler),
// then the NB recurrence steps run.  Callers use NB = 8 for full blocks and
// NB = 1 for remainders, so the hot loops are branch-free.
// ---------------------------------------------------------------------------

template <int G, int R, int NB>
__device__ __forceinline__ void fwd_block(const float (&fv)[NB], const float (&nu_hi)[G],
                                          const float (&nu_lo)[G], float dnu, const Casc& k,
                                          float (&v1)[4 * G], float (&v2)[4 * G],
                                          float (&y1)[4 * G], float (&y2)[4 * G],
                                          float* out_row, int out_stride) {
    float cc[NB][G], sn[NB][G];
#pragma unroll
    for (int q = 0; q < NB; ++q) phasors<G, R>(fv[q], nu_hi, nu_lo, dnu, cc[q], sn[q]);
#pragma unroll
    for (int q = 0; q < NB; ++q) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float u0 = cc[q][g], u1 = sn[q][g], u2 = fv[q] * cc[q][g], u3 = fv[q] * sn[q][g];
            const float o0 = cstep(u0, v1[4 * g + 0], v2[4 * g + 0], y1[4 * g + 0], y2[4 * g + 0], k);
            const float o1 = cstep(u1, v1[4 * g + 1], v2[4 * g + 1], y1[4 * g + 1], y2[4 * g + 1], k);
            const float o2 = cstep(u2, v1[4 * g + 2], v2[4 * g + 2], y1[4 * g + 2], y2[4 * g + 2], k);
            const float o3 = cstep(u3, v1[4 * g + 3], v2[4 * g + 3], y1[4 * g + 3], y2[4 * g + 3], k);
            if (out_row) {
                out_row[((4 * g + 0) * TILE + q) * out_stride] = o0;
                out_row[((4 * g + 1) * TILE + q) * out_stride] = o1;
                out_row[((4 * g + 2) * TILE + q) * out_stride] = o2;
                out_row[((4 * g + 3) * TILE + q) * out_stride] = o3;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Kernel arguments
// ---------------------------------------------------------------------------

struct TermDev {
    const float* nu_hi;  // [n] batch-relative
    const float* nu_lo;
    const float* w;
    float dnu;
    int n;       // terms in the batch
    int anchor;  // phasor anchor block (== G1); groups never straddle anchors
};

struct Pass1Args {
    const float* f;
    const float* fY;  // f tile-major (ty_index): a warp's 32-row segment is 4 KB contiguous
    int B, H, W;
    int Ey, nseg;  // y mirror extension; checkpoint segments per y-chunk
    int nyc, ych_rows, ywarm;  // y-chunks (at most ych_rows output rows each); warm-up rows (mult. of 32)
    int row0, row1;            // output rows of this call (equal chunks start at row0)
    // unequal chunks (ylpt, at most 3): rows [0, yb1), [yb1, yb2), [yb2, H);
    // scalars, not a table: a dynamically indexed parameter array made ptxas
    // spill in this kernel (9% slower pass 1 on config 5)
    int ylpt, yb1, yb2;
    int Ex, ne, edge_all, ntx;
    int nst;           // stripes of P1_WARPS column tiles (one pass-1 block each, per term)
    int st0, nst_run;  // stripes [st0, st0 + nst_run) in this launch
    int term0, nterm;  // terms [term0, term0 + nterm) of the batch in this launch
    int cs;            // stripes per thread-block cluster (1: no clusters; divides nst_run)
    int hq;            // zero unit (ZU launch): virtual rows = row quarters of 32-row segments
    int zyc, zrows;    // ... in y-chunks of zrows virtual rows
    Casc k;
    TermDev t;
    // Gaussian layouts (float4 = the 4 planes of one term, or the 4 states
    // (v1,v2,y1,y2) of one plane):
    float* ckpt;    // float4 [nseg][n][B][W][4 planes]
    float* floc;    // float4 [n][B][W][H]  tile-local forward along x (x-major)
                    //   (box: planar [n*4][B][W][H] y-filtered values)
    // x chain across stripes (decoupled hand-off, serial per (term, frame,
    // 32-row segment)): warp 0 of stripe s waits for stripe s-1's flag and
    // starts from mail slot s; warp 3 publishes its end state into slot s+1
    float* mail;           // float4 [n][B][nst+1][H][4 planes]; slot 0 unused (zero start at x = 0)
    int* flags;            // [n][B][nst][nsegH]: 1 once stripe s's slot s+1 rows of segment k are out
    int nsegH;             // ceil(H / 32)
    unsigned int* ticket;  // block dispatch counter (stripe-major order, see k_pass1_gauss)
    float* edge;    // float4 [n][B][ne][H] y-filtered values at x-edge columns
};

// Mirrored x-extensions (spatial.py:171 with pad = W-1 truncated to ext_x,
// _core.pyx:56-96) per (row, term), after pass 1: the forward state S0 at
// x = 0 (the left extension, which the pass-1 chain started from zero) and
// the backward start state at x = W-1 (the right extension, in closed form).
struct EdgeArgs {
    int B, H, W;
    int row0, row1;       // rows of this call
    int Ex, ne, edge_all, nst;  // nst = stripes (mail slot nst = chain end state at x = W)
    Casc k;
    int n;                // terms in the batch
    const float* edge;    // float4 [n][B][ne][H]
    const float* mail;    // chain end states: slot ntx = forward state at x = W of the zero-start chain
    float MW[16];         // zero-input state transfer over W samples (column-major)
    float Rx[16];         // right extension: bstate = Rx . s(W) + sum_e bx[e] Y(W-2-e)
    const float4* bx;     // [Ex] (see right_ext_coeffs)
    float* s0;            // float4 [n][B][H][4 planes] left-extension state S0
    float* bstate;        // float4 [n][B][H][4 planes] backward start state
};

struct Pass2Args {
    const float* fT;  // [B][W][H]
    int B, H, W, ntx;
    Casc k;
    TermDev t;
    int ngroups;       // ceil((t.n - term0) / G2)
    int term0;         // first term of the batch in this launch
    float wscale;      // g^2: undoes the two pure x sweeps (1 for box)
    int rb0, nrb_run;     // 128-row blocks [rb0, rb0 + nrb_run) in this launch
    int tiles_per_chunk;  // x-chunking of rows (gauss); == ntx for one chunk
    // unequal x-chunks (xlpt, at most 3): tiles [0, xb1), [xb1, xb2), [xb2, ntx),
    // dispatched in the order packed in xord (2 bits per rank, costliest
    // first); scalars rather than tables (dynamically indexed parameter
    // arrays cost registers)
    int xlpt, xb1, xb2, xord;
    int warm_tiles;       // warm-up tiles of a chunk's backward sweep
    const float* floc;    // forward output of the zero-start chain (exact once corrected)
    // exact forward = floc + Hx[x] . S0 for x < nHx (the response to the
    // left-extension state decays below 1e-9 relative beyond nHx)
    int nHx;
    const float4* Hx;     // [nHx] zero-input cascade output at x from unit states at x = 0
    const float* s0;      // float4 [n][B][H][4]
    const float* bstate;  // float4 [n][B][H][4]
    float* part;          // [ngroups*2][B][W][H]
    int order;            // k_pass2_gr block order (TBF_OPT_P2_ORDER)
};

struct ReduceArgs {
    const float* part;  // [ngroups*2][B][W][H]
    int ngroups;
    int B, H, W;
    const float* in_num;  // [B][H][W] added to the partials when non-null
    const float* in_den;
    float* num;           // [B][H][W] written when non-null
    float* den;
    const float* f;       // guard fallback (when out != null)
    float* out;           // [B][H][W] guarded ratio when non-null
    unsigned long long* counters;
    int i_base;           // first row of this launch (multiple of RED_I)
    const float* zpart;   // zero unit's num plane (x-major) added last when non-null
    float den_add;        // ... with its den, w0 exactly (engines.py:270)
};

// Pass 2 of the zero unit (k_pass2_zero): the x backward of its four row
// quarters and num at the image rows; den is w0, added by the reduce.
struct ZeroArgs {
    int B, H, W, ntx, hq;
    int term;             // the unit's term slot in the batch
    Casc k;
    int tiles_per_chunk, warm_tiles;
    float wt;             // w0 * wscale
    const float* floc;
    int nHx;
    const float4* Hx;
    const float* s0;
    const float* bstate;
    float* num;           // x-major plane (xm_index) of image rows
};

// ---------------------------------------------------------------------------
// Pass 1 (recursive Gaussian): y-direction forward/backward + x tile-local
// forward.  Replaces smooth_plane's first 1-D pass (spatial.py:169-170,
// _core.pyx:56-96) for the 4 auxiliary planes of one term, fused with their
// generation (engines.py:272-287).  One warp = 32 columns x 1 term.
// ---------------------------------------------------------------------------

__device__ __forceinline__ float4 f4(float a, float b, float c, float d) {
    return make_float4(a, b, c, d);
}

// 8 samples of the forward sweep of one term (phasors first, then the 4
// plane recurrences); optionally store outputs into the smem segment tile.
template <bool STORE>
__device__ __forceinline__ void p1_fwd8(const float (&fv)[8], float nu_hi, float nu_lo,
                                        const Casc& k, float (&v1)[4], float (&v2)[4],
                                        float (&y1)[4], float (&y2)[4], float4* row, bool st = true) {
    float cs[8], sn[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) sincos_fma(phase(nu_hi, nu_lo, fv[q]), &sn[q], &cs[q]);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float u[4] = {cs[q], sn[q], fv[q] * cs[q], fv[q] * sn[q]};
        float o[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) o[p] = cstep(u[p], v1[p], v2[p], y1[p], y2[p], k);
        if (STORE && st) row[q * BUF_LD] = make_float4(o[0], o[1], o[2], o[3]);
    }
}

// FOLD: the g^2 that undoes the two pure y sweeps is folded into the pass-2
// weights (g^4 there) instead of one multiply per plane-sample here; used when
// T/g^4 stays far from the fp32 range limit.
// LPT: unequal y-chunks (ylpt/yb1/yb2); the equal-chunk instantiation keeps
// the chunk arithmetic rematerialisable (no extra live registers)
// MODE: 0 one y-chunk per column (the original code paths), 1 equal y-chunks
// (interior chunks' warm-up rows read as whole fY tiles), 2 planned unequal
// chunks (LPT bounds + the same warm-up reads).  Separate instantiations keep
// each one's register allocation: the warm-up fast path cost config 3 (one
// chunk) 0.8% through register pressure while gaining 2.5% on config 2.
// ZU: the zero-frequency term as one packed unit (engines.py:
// 265-271): nu = 0 needs only F[f] (den += w0 exactly), so the unit's four
// float4 lanes carry f itself at four row quarters (virtual row v, plane p =
// image row v + p*hq) instead of (cos, sin, f cos, f sin) of one row: a
// quarter of a term's sweeps and bytes.  Plane 0 starts at the exact mirror
// extension, planes 1-3 a decay length Ey >= K above their quarter (rows of
// the image), plane 3 runs on past the image into a general reflection that
// the backward start forgets within K.
template <bool FOLD, int MODE, bool ZU = false>
__global__ void __launch_bounds__(P1_WARPS * 32, P1_BLOCKS_PER_SM) k_pass1_gauss(const __grid_constant__ Pass1Args a) {
    constexpr bool LPT = MODE == 2;
    extern __shared__ float smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    __shared__ unsigned int s_ticket;
    // one block = one term x one stripe of P1_WARPS column tiles (warp w =
    // tile w of the stripe).  Dispatch order from a ticket taken at block
    // start (not blockIdx: the x chain makes stripe s wait for stripe s-1, so
    // every block a block waits for must have been dispatched before it).
    // Stripe slowest, then frame, y-chunk, term fastest: the blocks sharing a
    // stripe's f run together, and a wave spreads over many independent
    // chains (the hand-off lag of a wave grows with the stripes of one chain
    // in it).
    // clusters of a.cs consecutive stripes (a.cs > 1): the cluster's first
    // block takes the ticket, the others read it through DSMEM; each block's
    // incoming hand-off slot and its FULL / EMPTY mbarriers are set up first
    __shared__ __align__(8) uint64_t s_full, s_empty;
    const unsigned crank = a.cs > 1 ? cluster_ctarank() : 0u;
    if (threadIdx.x == 0) {
        if (crank == 0) s_ticket = atomicAdd(a.ticket, 1u);
        if (a.cs > 1) {
            mbar_init_cta(&s_full, 32);
            mbar_init_cta(&s_empty, 32);
            fence_mbar_init();
        }
    }
    if (a.cs > 1) {
        cluster_sync_all();
        if (threadIdx.x == 0 && crank != 0) s_ticket = ld_cluster_u32(map_cluster(smem_addr(&s_ticket), 0));
    }
    __syncthreads();
    // a programmatically dependent next launch (the next host strip) may
    // start once every block of this one has got here
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    int term, stripe_r, chunk, b;
    {
        unsigned int idx = s_ticket;
        if (ZU) {  // one term; y-chunks of the virtual rows
            term = a.term0;
            chunk = (int)(idx % (unsigned)a.zyc);
            idx /= (unsigned)a.zyc;
        } else {
            term = a.term0 + (int)(idx % (unsigned)a.nterm);
            idx /= (unsigned)a.nterm;
            chunk = (int)(idx % (unsigned)a.nyc);
            idx /= (unsigned)a.nyc;
        }
        b = (int)(idx % (unsigned)a.B);
        stripe_r = (int)(idx / (unsigned)a.B) * a.cs + (int)crank;
    }
    const int H = a.H, W = a.W;
    const int stripe = a.st0 + stripe_r;
    const int tile_x = stripe * P1_WARPS + warp;
    const int x0 = tile_x * TILE;
    const int x = x0 + lane;
    const bool xv = x < W;
    const int xc = xv ? x : W - 1;
    // the last stripe's warps past the image edge (tlen <= 0) run clamped
    // columns without storing anything: every warp takes part in the hand-off
    const int tlen = min(TILE, W - x0);
    // segment tile [row][col] of float4 (the 4 planes of a pixel adjacent),
    // padded row stride BUF_LD: column access (phases A/B) is contiguous, row
    // access (epilogue) hits 4 distinct bank groups -> 4 wavefronts, optimal
    float4* const buf = reinterpret_cast<float4*>(smem) + (size_t)warp * TILE * BUF_LD;
    float4* const bl = buf + lane;           // own column (phases A/B)
    float4* const br = buf + lane * BUF_LD;  // own row (epilogue)
    const float nu_hi = ZU ? 0.f : a.t.nu_hi[term], nu_lo = ZU ? 0.f : a.t.nu_lo[term];
    const Casc k = a.k;
    const int Ey = a.Ey;
    const int iend = H + Ey;  // forward runs over extended rows [-Ey, H+Ey)
    // this lane's column (clamped to the image) of the tile-major copy at
    // image row r >= 0: unsigned index math (cheaper than ty_index's signed
    // division), recomputed from parameters each time rather than hoisted (a
    // hoisted base + stride stays live through the kernel and made ptxas spill)
    const size_t tstr = (size_t)((W + TILE - 1) / TILE) * TILE * TILE;  // floats per 32-row tile row
    auto frow = [&](int r) -> const float* {
        const unsigned ur = (unsigned)r, ux = (unsigned)xc;
        const unsigned nys = ((unsigned)H + 31u) >> 5;
        return a.fY + ((size_t)b * nys + (ur >> 5)) * tstr + (ux >> 5) * 1024u + (ur & 31u) * 32u + (ux & 31u);
    };
    auto fload = [&](int i) -> float {  // f at extended row i (mirrored), clamped
        i = max(-Ey, min(i, iend - 1));
        if (MODE == 0) return __ldg(a.fY + ty_index(b, xc, mirror1(i, H), W, H));
        return __ldg(frow(mirror1(i, H)));
    };
    // the four plane inputs at (extended / virtual) row i
    auto modrow = [&](int i, float (&u)[4]) {
        if (ZU) {  // rows i + p*hq of the image, one reflection at either end
#pragma unroll
            for (int p = 0; p < 4; ++p) u[p] = __ldg(frow(mirror1(i + p * a.hq, H)));
        } else {
            const float fs = fload(i);
            float s0, c0;
            sincos_fma(phase(nu_hi, nu_lo, fs), &s0, &c0);
            u[0] = c0;
            u[1] = s0;
            u[2] = fs * c0;
            u[3] = fs * s0;
        }
    };
    // y-chunk: output rows [R0, R1).  The forward sweep starts at A0 = R0 -
    // ywarm from a steady-state guess (exact -Ey start for the top chunk); the
    // backward starts at Bend = R1 + ywarm (exact H+Ey end for the bottom
    // chunk).  ywarm >= the decay length K, so guesses fade below eps.
    int R0, R1;
    if (ZU) {
        R0 = chunk * a.zrows;
        R1 = min(a.hq, R0 + a.zrows);
    } else if (LPT) {
        R0 = chunk == 0 ? 0 : (chunk == 1 ? a.yb1 : a.yb2);
        R1 = chunk == 0 ? a.yb1 : (chunk == 1 ? a.yb2 : H);
    } else {
        R0 = a.row0 + chunk * a.ych_rows;
        R1 = min(a.row1, R0 + a.ych_rows);
    }
    const int A0 = R0 - a.ywarm <= 0 ? -Ey : R0 - a.ywarm;
    const int Bend = ZU ? (R1 + a.ywarm >= a.hq + Ey ? a.hq + Ey : R1 + a.ywarm)
                        : (R1 + a.ywarm >= iend ? iend : R1 + a.ywarm);
    // checkpoints: float4 per plane, [chunk*nseg + local seg][term][b][x][4]
    const size_t cks = (size_t)a.t.n * a.B * W * 4;  // float4 stride between segments
    float4* const ck0 = reinterpret_cast<float4*>(a.ckpt) +
                        (((size_t)term * a.B + b) * W + xc) * 4 + (size_t)chunk * a.nseg * cks;

    float v1[4], v2[4], y1[4], y2[4];
    {
        float u[4];
        modrow(A0, u);
#pragma unroll
        for (int p = 0; p < 4; ++p) csteady(u[p], v1[p], v2[p], y1[p], y2[p], k);
    }

    // ---- phase A: forward sweep, double-buffered 8-row blocks ----
    auto step1 = [&](int i) {
        float u[4];
        modrow(i, u);
#pragma unroll
        for (int p = 0; p < 4; ++p) cstep(u[p], v1[p], v2[p], y1[p], y2[p], k);
    };
    if (ZU) {  // lead-in in 8-row blocks, the next block's loads in flight
        float cur[8][4], nxt[8][4];
        int i = A0;
        for (; i < A0 + ((R0 - A0) & 7); ++i) step1(i);
#pragma unroll
        for (int q = 0; q < 8; ++q) modrow(i + q, cur[q]);
#pragma unroll 1
        for (; i < R0; i += 8) {
#pragma unroll
            for (int q = 0; q < 8; ++q) modrow(i + 8 + q, nxt[q]);
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
                for (int p = 0; p < 4; ++p) cstep(cur[q][p], v1[p], v2[p], y1[p], y2[p], k);
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
                for (int p = 0; p < 4; ++p) cur[q][p] = nxt[q][p];
        }
    } else if (MODE > 0 && A0 >= 0) {
        // interior chunk: the warm-up rows [A0, R0) are whole 32-row tiles of
        // fY (both multiples of 32): 8-row blocks at immediate offsets, one
        // pointer step per block instead of a mirrored, clamped index per row
        const float* p = frow(A0);
        float cur[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) cur[q] = ldg_pinned(p + q * 32);
#pragma unroll 1
        for (int i = A0; i < R0; i += 8) {
            const float* pn = ((i + 8) & 31) ? p + 8 * 32 : p - 24 * 32 + tstr;
            if (i + 8 >= R0) pn = p;  // last block: (re)load a valid address
            float nx[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) nx[q] = ldg_pinned(pn + q * 32);
            p1_fwd8<false>(cur, nu_hi, nu_lo, k, v1, v2, y1, y2, nullptr);
#pragma unroll
            for (int q = 0; q < 8; ++q) cur[q] = nx[q];
            p = pn;
        }
    } else {
        int i = A0;
        for (; i < A0 + ((R0 - A0) & 7); ++i) step1(i);  // remainder of the lead-in rows
        float cur[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) cur[q] = fload(i + q);
#pragma unroll 1
        for (; i < R0; i += 8) {  // rest of the lead-in (mirror extension / warm-up), ends at R0
            float nx[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) nx[q] = fload(i + 8 + q);
            p1_fwd8<false>(cur, nu_hi, nu_lo, k, v1, v2, y1, y2, nullptr);
#pragma unroll
            for (int q = 0; q < 8; ++q) cur[q] = nx[q];
        }
    }

    // ---- phases A and B as one loop over 2*nseg steps: steps 0..nseg-1 are
    // the forward sweep top->bottom (checkpoint stores), steps nseg..2nseg-1
    // revisit the segments bottom->top (restore, forward recompute into the
    // smem tile, backward, epilogue).  Both phases share one copy of the
    // forward code (instruction-cache footprint); phase A's tile stores are
    // predicated off except on its last step (tile_st below).  f and
    // checkpoints are prefetched one step ahead.
    float p1[4], p2[4], q1[4], q2[4];
    // F_loc layout: float4 [term][b][row block of 32][x][32 rows] (row-block
    // tiled so a pass-2 warp streams its rows contiguously along x)
    const int nrbk = (H + FL_RB - 1) / FL_RB;
    float4* const fl0 = reinterpret_cast<float4*>(a.floc) + ((size_t)term * a.B + b) * nrbk * W * (size_t)FL_RB;
    float4* const ed0 = reinterpret_cast<float4*>(a.edge) + ((size_t)term * a.B + b) * a.ne * (size_t)H;
    // x chain across stripes: mail slot s = state at stripe s's start
    float4* const mail0 = reinterpret_cast<float4*>(a.mail) +
                          (((size_t)term * a.B + b) * (a.nst + 1) + stripe) * (size_t)H * 4;
    int* const flag0 = a.flags + (((size_t)term * a.B + b) * a.nst + stripe) * a.nsegH;
    // hand-off slots between the stripe's warps: slot w (warp w -> w+1) holds
    // one float4 per plane and row, after the P1_WARPS tiles
    float4* const hand = reinterpret_cast<float4*>(smem) + (size_t)P1_WARPS * TILE * BUF_LD;
    // incoming slot of a cluster hand-off (written remotely by the previous
    // stripe's last warp); in DSMEM terms, the next block's slot for ours
    float4* const hand_in = hand + (size_t)(P1_WARPS - 1) * 4 * TILE;
    const bool cl_in = a.cs > 1 && crank > 0;                    // hand-off in from the cluster
    const bool cl_out = a.cs > 1 && crank + 1 < (unsigned)a.cs;  // hand-off out to the cluster
    const uint32_t next_slot = cl_out ? map_cluster(smem_addr(hand_in), crank + 1) : 0u;
    const uint32_t next_full = cl_out ? map_cluster(smem_addr(&s_full), crank + 1) : 0u;
    const uint32_t prev_empty = cl_in ? map_cluster(smem_addr(&s_empty), crank - 1) : 0u;
    int nout = 0;  // output segments done (the hand-off barriers pair up per segment)
    const int nseg = (Bend - R0 + TILE - 1) / TILE;  // local segments of this chunk
    const int nsteps = 2 * nseg;
    float seg_f[TILE];
    if (!ZU) {
#pragma unroll
        for (int q = 0; q < TILE; ++q) seg_f[q] = fload(R0 + q);
    }
#pragma unroll 1
    for (int step = 0; step < nsteps; ++step) {
        const bool phaseB = step >= nseg;
        const int seg = phaseB ? nsteps - 1 - step : step;
        const int i0 = R0 + seg * TILE;
        const int len = min(TILE, Bend - i0);
        if (!phaseB && xv) {
            float4* ck = ck0 + (size_t)seg * cks;
#pragma unroll
            for (int p = 0; p < 4; ++p) ck[p] = f4(v1[p], v2[p], y1[p], y2[p]);
        }
        // the next step's segment: its f rows are loaded during this step's
        // forward (in-place refill below), its checkpoint (phase B) after it
        const int ns = step + 1 < nseg ? step + 1 : max(nsteps - 2 - step, 0);
        const int rn = R0 + ns * TILE;
        const bool nfast = !ZU && rn >= 0 && rn + TILE <= H;  // next segment: one whole fY tile
        const bool full = !ZU && step != nseg && len == TILE;
        // forward over the segment into the smem tile (own column), 4 x 8
        // samples; the first phase-B step finds the tile already filled by the
        // last phase-A step.  In-place refill: after each 8-row block has
        // consumed its rows, the same registers take the next segment's rows
        // (a whole step ahead of their use).  Measured 1-2% faster on configs
        // 1-4 than a separate prefetch array copied at the end of each step.
        const float* const fpn = MODE == 0 ? a.fY + ty_index(b, x0 + lane, nfast ? rn : 0, W, H) : frow(nfast ? rn : 0);
        // phase A's forward outputs are not needed except on its last step
        // (the first phase-B step reuses that tile): no shared-memory stores
        // otherwise (the L1/shared pipe runs at ~80% of peak in this kernel)
        const bool tile_st = TBF_P1_ASTORE || phaseB || step == nseg - 1;
        if (full) {
#pragma unroll
            for (int q0 = 0; q0 < TILE; q0 += 8) {
                p1_fwd8<true>(*reinterpret_cast<const float(*)[8]>(&seg_f[q0]), nu_hi, nu_lo, k, v1, v2,
                              y1, y2, bl + q0 * BUF_LD, tile_st);
                if (nfast) {
#pragma unroll
                    for (int q = q0; q < q0 + 8; ++q) seg_f[q] = ldg_pinned(fpn + q * 32);
                }
            }
        } else if (ZU) {
            if (step != nseg) {
                // 8-row blocks, the next block's 32 loads in flight meanwhile
                float cur[8][4], nxt[8][4];
#pragma unroll
                for (int q = 0; q < 8; ++q) modrow(i0 + q, cur[q]);
#pragma unroll 1
                for (int r0 = 0; r0 < len; r0 += 8) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) modrow(min(i0 + r0 + 8 + q, Bend - 1), nxt[q]);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (r0 + q < len) {
                            float o[4];
#pragma unroll
                            for (int p = 0; p < 4; ++p) o[p] = cstep(cur[q][p], v1[p], v2[p], y1[p], y2[p], k);
                            bl[(r0 + q) * BUF_LD] = make_float4(o[0], o[1], o[2], o[3]);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q)
#pragma unroll
                        for (int p = 0; p < 4; ++p) cur[q][p] = nxt[q][p];
                }
            }
        } else {
            if (step != nseg) {
                for (int r = 0; r < len; ++r) {
                    float u[4];
                    modrow(i0 + r, u);
                    float o[4];
#pragma unroll
                    for (int p = 0; p < 4; ++p) o[p] = cstep(u[p], v1[p], v2[p], y1[p], y2[p], k);
                    bl[r * BUF_LD] = make_float4(o[0], o[1], o[2], o[3]);
                }
            }
            if (nfast) {
#pragma unroll
                for (int q = 0; q < TILE; ++q) seg_f[q] = ldg_pinned(fpn + q * 32);
            }
        }
        if (!ZU && !nfast) {  // boundary segments (mirror extension): generic loads
#pragma unroll
            for (int q = 0; q < TILE; ++q) seg_f[q] = fload(rn + q);
        }
        if (!phaseB) continue;
        if (step + 1 < nsteps) {
            // the next step's forward restarts from its segment's checkpoint:
            // loaded straight into the forward state, which this step no
            // longer needs, a whole backward + epilogue ahead of its use (no
            // prefetch registers and restore moves)
            const float4* ck = ck0 + (size_t)ns * cks;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const float4 c = ck[p];
                v1[p] = c.x;
                v2[p] = c.y;
                y1[p] = c.z;
                y2[p] = c.w;
            }
        }
        if (seg == nseg - 1) {
            // backward start = steady state of the last forward output (_core.pyx:85-87)
            const float4 lastf = bl[(len - 1) * BUF_LD];
            const float lf[4] = {lastf.x, lastf.y, lastf.z, lastf.w};
#pragma unroll
            for (int p = 0; p < 4; ++p) csteady(lf[p], p1[p], p2[p], q1[p], q2[p], k);
        }
        // backward sweep over the segment, in place
        if (len == TILE) {
#pragma unroll 1
            for (int r0 = TILE - 1; r0 >= 0; r0 -= 8) {
                float4* row = bl + r0 * BUF_LD;
                float4 in[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) in[q] = row[-q * BUF_LD];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float iv4[4] = {in[q].x, in[q].y, in[q].z, in[q].w};
                    float o[4];
#pragma unroll
                    for (int p = 0; p < 4; ++p) o[p] = cstep(iv4[p], p1[p], p2[p], q1[p], q2[p], k);
                    row[-q * BUF_LD] = make_float4(o[0], o[1], o[2], o[3]);
                }
            }
        } else {
            for (int r = len - 1; r >= 0; --r) {
                const float4 c4 = bl[r * BUF_LD];
                const float iv4[4] = {c4.x, c4.y, c4.z, c4.w};
                float o[4];
#pragma unroll
                for (int p = 0; p < 4; ++p) o[p] = cstep(iv4[p], p1[p], p2[p], q1[p], q2[p], k);
                bl[r * BUF_LD] = make_float4(o[0], o[1], o[2], o[3]);
            }
        }
        if (i0 >= R1) continue;  // warm-up / extension segment: no output
        __syncwarp();
        // epilogue: lane <-> row i; forward along x over the tile's 32
        // columns, starting from the state at the tile's first column: from
        // the warp to the left through smem (named barriers per link w ->
        // w+1: FULL 1 + w when the slot is written, EMPTY 1 + P1_WARPS + w
        // when it has been read), for warp 0 from stripe s-1 through the L2
        // mailbox and its flag (zero at x = 0: pass 2 adds the response to
        // the left extension's state).
        const int i = i0 + lane;
        const bool rowv = lane < min(len, R1 - i0);
        const bool last_out = i0 == R0;  // segments run bottom to top
        float lv1[4], lv2[4], ly1[4], ly2[4];
        if (warp > 0) {
            named_bar_sync(1 + (warp - 1), 64);
            const float4* hs = hand + ((size_t)(warp - 1) * 4) * TILE + lane;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const float4 c = hs[p * TILE];
                lv1[p] = c.x;
                lv2[p] = c.y;
                ly1[p] = c.z;
                ly2[p] = c.w;
            }
            if (!last_out) named_bar_arrive(1 + P1_WARPS + (warp - 1), 64);
        } else if (cl_in) {
            // the previous stripe of the cluster wrote our slot (DSMEM)
            mbar_wait_cluster(&s_full, (unsigned)nout & 1u);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const float4 c = hand_in[p * TILE + lane];
                lv1[p] = c.x;
                lv2[p] = c.y;
                ly1[p] = c.z;
                ly2[p] = c.w;
            }
            if (!last_out) mbar_arrive_remote(prev_empty);  // slot free for its next segment
        } else if (stripe > 0) {
            // stripe s-1 hands its end state over: wait for its flag for this
            // segment (a hand-off never arrives only if the dispatch order
            // were broken: fail the launch after ~10 s instead of hanging)
            const int* pf = flag0 - a.nsegH + (i0 >> 5);
            unsigned int spins = 0;
            while (ld_relaxed(pf) == 0) {
                __nanosleep(32);
                if (++spins == (1u << 27)) __trap();
            }
            const float4* mb = mail0 + (size_t)i * 4;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const float4 c = rowv ? ld_relaxed4(mb + p) : f4(0.f, 0.f, 0.f, 0.f);
                lv1[p] = c.x;
                lv2[p] = c.y;
                ly1[p] = c.z;
                ly2[p] = c.w;
            }
        } else {
#pragma unroll
            for (int p = 0; p < 4; ++p) lv1[p] = lv2[p] = ly1[p] = ly2[p] = 0.f;
        }
        float4* const fl = fl0 + ((size_t)(i / FL_RB) * W + x0) * FL_RB + (i % FL_RB);
        if (rowv && tlen > 0) {
            const bool edge_tile = a.edge_all || x0 <= a.Ex || x0 + tlen - 1 >= W - 1 - a.Ex;
            if (tlen == TILE && !edge_tile) {
#pragma unroll 1
                for (int xb = 0; xb < TILE; xb += 8) {
                    float yv[8][4];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float4 t4 = br[xb + q];
                        const float sc = FOLD ? 1.f : k.gg;
                        yv[q][0] = FOLD ? t4.x : t4.x * sc;
                        yv[q][1] = FOLD ? t4.y : t4.y * sc;
                        yv[q][2] = FOLD ? t4.z : t4.z * sc;
                        yv[q][3] = FOLD ? t4.w : t4.w * sc;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float o[4];
#pragma unroll
                        for (int p = 0; p < 4; ++p) o[p] = cstep(yv[q][p], lv1[p], lv2[p], ly1[p], ly2[p], k);
                        st_stream(fl + (size_t)(xb + q) * FL_RB, f4(o[0], o[1], o[2], o[3]));
                    }
                }
            } else {
                for (int xx = 0; xx < tlen; ++xx) {
                    const int gx = x0 + xx;
                    const float4 t4 = br[xx];
                    // undo the 1/g^2 of the two pure y sweeps
                    const float sc = FOLD ? 1.f : k.gg;
                    const float yv[4] = {t4.x * sc, t4.y * sc, t4.z * sc, t4.w * sc};
                    float o[4];
#pragma unroll
                    for (int p = 0; p < 4; ++p) o[p] = cstep(yv[p], lv1[p], lv2[p], ly1[p], ly2[p], k);
                    st_stream(fl + (size_t)xx * FL_RB, f4(o[0], o[1], o[2], o[3]));
                    if (a.edge_all || gx <= a.Ex || gx >= W - 1 - a.Ex) {
                        const int e = a.edge_all ? gx : (gx <= a.Ex ? gx : gx - (W - 1 - a.Ex) + a.Ex + 1);
                        ed0[(size_t)e * H + i] = f4(yv[0], yv[1], yv[2], yv[3]);
                    }
                }
            }
        }
        if (warp < P1_WARPS - 1) {
            if (nout > 0) named_bar_sync(1 + P1_WARPS + warp, 64);  // the slot's previous state was read
            float4* hs = hand + ((size_t)warp * 4) * TILE + lane;
#pragma unroll
            for (int p = 0; p < 4; ++p) hs[p * TILE] = f4(lv1[p], lv2[p], ly1[p], ly2[p]);
            named_bar_arrive(1 + warp, 64);
        } else if (cl_out) {
            // to the next stripe of the cluster: its slot (DSMEM) once it read
            // the previous segment's, then its FULL barrier (release)
            if (nout > 0) mbar_wait_cluster(&s_empty, (unsigned)(nout - 1) & 1u);
#pragma unroll
            for (int p = 0; p < 4; ++p)
                st_cluster4(next_slot + (uint32_t)((p * TILE + lane) * 16), f4(lv1[p], lv2[p], ly1[p], ly2[p]));
            mbar_arrive_remote(next_full);
        } else {
            // the stripe's end state (clamped warps past the image edge pass
            // the state of its last column through unchanged) to mail slot
            // s+1 (L2), then the flag: every lane releases its own stores
            if (rowv) {
                float4* mb = mail0 + ((size_t)H + i) * 4;
#pragma unroll
                for (int p = 0; p < 4; ++p) __stcg(mb + p, f4(lv1[p], lv2[p], ly1[p], ly2[p]));
            }
            st_release(flag0 + (i0 >> 5), 1);
        }
        ++nout;
        __syncwarp();
    }
    // a cluster's blocks keep their shared memory until every remote access
    // to it is done
    if (a.cs > 1) cluster_sync_all();
}

// ---------------------------------------------------------------------------
// Edge: per (row, term) the mirrored x-extensions (spatial.py:171 with pad =
// W-1 truncated to ext_x, _core.pyx:56-96) from the edge columns pass 1
// wrote: the left extension's forward state S0 at x = 0 (the pass-1 chain
// started from zero; pass 2 adds the response to S0) and the backward start
// state at x = W-1 (right extension in closed form).
// ---------------------------------------------------------------------------

__device__ __forceinline__ void cstep4(const float4& u, float (&v1)[4], float (&v2)[4],
                                       float (&y1)[4], float (&y2)[4], const Casc& k,
                                       float (&o)[4]) {
    o[0] = cstep(u.x, v1[0], v2[0], y1[0], y2[0], k);
    o[1] = cstep(u.y, v1[1], v2[1], y1[1], y2[1], k);
    o[2] = cstep(u.z, v1[2], v2[2], y1[2], y2[2], k);
    o[3] = cstep(u.w, v1[3], v2[3], y1[3], y2[3], k);
}

__global__ void __launch_bounds__(128) k_edge(const __grid_constant__ EdgeArgs a) {
    const int i = a.row0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.row1) return;
    const int bt = blockIdx.y;  // term * B + b
    const int H = a.H, W = a.W, Ex = a.Ex;
    const Casc k = a.k;
    const float4* ed = reinterpret_cast<const float4*>(a.edge) + (size_t)bt * a.ne * H + i;
    auto eidx = [&](int xx) -> int {
        return a.edge_all ? xx : (xx <= Ex ? xx : xx - (W - 1 - Ex) + Ex + 1);
    };
    float v1[4], v2[4], y1[4], y2[4], o[4];
    {
        const float4 u = ed[(size_t)eidx(Ex) * H];  // mirror(-Ex)
        csteady(u.x, v1[0], v2[0], y1[0], y2[0], k);
        csteady(u.y, v1[1], v2[1], y1[1], y2[1], k);
        csteady(u.z, v1[2], v2[2], y1[2], y2[2], k);
        csteady(u.w, v1[3], v2[3], y1[3], y2[3], k);
    }
    // left extension x = -Ex..-1 reads Y(-x); 8 loads in flight
    for (int xb = -Ex; xb < 0; xb += 8) {
        float4 u[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) u[q] = ed[(size_t)eidx(max(1, -(xb + q))) * H];
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (xb + q < 0) cstep4(u[q], v1, v2, y1, y2, k, o);
    }
    float4* s0 = reinterpret_cast<float4*>(a.s0) + ((size_t)bt * H + i) * 4;
#pragma unroll
    for (int p = 0; p < 4; ++p) s0[p] = f4(v1[p], v2[p], y1[p], y2[p]);
    // forward state at x = W: the zero-start chain's end state plus the
    // response to S0 carried over the W samples
    const float4* cw = reinterpret_cast<const float4*>(a.mail) + (((size_t)bt * (a.nst + 1) + a.nst) * H + i) * 4;
    float s[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float4 c = cw[p];
        const float z[4] = {v1[p], v2[p], y1[p], y2[p]};
        const float cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int r = 0; r < 4; ++r)
            s[p][r] = fmaf(a.MW[r], z[0], fmaf(a.MW[4 + r], z[1], fmaf(a.MW[8 + r], z[2], fmaf(a.MW[12 + r], z[3], cc[r]))));
    }
    // right extension (forward over x = W .. W-1+Ex on Y(2(W-1)-x), steady
    // start from its last output, backward back to x = W-1) in closed form:
    // the map is linear in the state at x = W and the Ex mirrored inputs
    float p1[4], p2[4], q1[4], q2[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float s0v = s[p][0], s1 = s[p][1], s2 = s[p][2], s3 = s[p][3];
        p1[p] = fmaf(a.Rx[0], s0v, fmaf(a.Rx[4], s1, fmaf(a.Rx[8], s2, a.Rx[12] * s3)));
        p2[p] = fmaf(a.Rx[1], s0v, fmaf(a.Rx[5], s1, fmaf(a.Rx[9], s2, a.Rx[13] * s3)));
        q1[p] = fmaf(a.Rx[2], s0v, fmaf(a.Rx[6], s1, fmaf(a.Rx[10], s2, a.Rx[14] * s3)));
        q2[p] = fmaf(a.Rx[3], s0v, fmaf(a.Rx[7], s1, fmaf(a.Rx[11], s2, a.Rx[15] * s3)));
    }
    for (int eb = 0; eb < Ex; eb += 8) {
        float4 u[8], c[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = min(eb + q, Ex - 1);
            u[q] = ed[(size_t)eidx(max(0, W - 2 - e)) * H];
            c[q] = __ldg(a.bx + e);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (eb + q < Ex) {
                const float uv[4] = {u[q].x, u[q].y, u[q].z, u[q].w};
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    p1[p] = fmaf(c[q].x, uv[p], p1[p]);
                    p2[p] = fmaf(c[q].y, uv[p], p2[p]);
                    q1[p] = fmaf(c[q].z, uv[p], q1[p]);
                    q2[p] = fmaf(c[q].w, uv[p], q2[p]);
                }
            }
        }
    }
    float4* bs = reinterpret_cast<float4*>(a.bstate) + ((size_t)bt * H + i) * 4;
#pragma unroll
    for (int p = 0; p < 4; ++p) bs[p] = f4(p1[p], p2[p], q1[p], q2[p]);
}

// ---------------------------------------------------------------------------
// Pass 2 (recursive Gaussian): x-direction backward sweep on the exact forward
// output, fused with demodulation + accumulation (engines.py:297-298).  One
// thread = one row x G terms.  Pass 1 wrote the forward output of a chain
// that started from zero at x = 0; the tiles with x < nHx add the response
// Hx[x] . S0 to the left-extension state (CORR instantiation).
// ---------------------------------------------------------------------------

template <int G>
struct P2Ctx {
    const float4* fl[G];  // this row, x = 0, per term
    const float* fT;
    const float4* s0[G];  // left-extension state S0, this row, per term
    float nu_hi[G], nu_lo[G], wt[G];
};

// Loads of one 4-step block (x = x0+m, m = mb, mb-1, .., mb-3; clamped).
template <int G, bool OUT>
__device__ __forceinline__ void p2_load4(const P2Ctx<G>& c, int x0, int mb, float4 (&fo)[4][G],
                                         float (&fv)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const size_t off = (size_t)(x0 + max(mb - q, 0)) * FL_RB;
#pragma unroll
        for (int g = 0; g < G; ++g) fo[q][g] = ld_stream(c.fl[g] + off);
        if (OUT) fv[q] = c.fT[off];
    }
}

// Exact forward output of plane p at x: floc + Hx[x] . S0 when CORR.
template <bool CORR>
__device__ __forceinline__ float p2_fwd(float fin, const float4& h, const float (&S)[4]) {
    if (!CORR) return fin;
    float F = fmaf(h.x, S[0], fin);
    F = fmaf(h.y, S[1], F);
    F = fmaf(h.z, S[2], F);
    return fmaf(h.w, S[3], F);
}

template <int G, bool OUT, bool CORR, bool SM = false>
__device__ __forceinline__ void p2_step4(const Pass2Args& a, const P2Ctx<G>& c, int x0, int mb,
                                         bool full, const float4 (&fo)[4][G], const float (&fv)[4],
                                         const float (&S)[G][4][4], float (&p1)[G][4],
                                         float (&p2)[G][4], float (&q1)[G][4], float (&q2)[G][4],
                                         float* pn, float* pd, bool iv, float2* sb = nullptr) {
    const Casc k = a.k;
    float cs[4][G], sn[4][G];
    if (OUT) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int g = 0; g < G; ++g)
                sincos_fma(phase(c.nu_hi[g], c.nu_lo[g], fv[q]), &sn[q][g], &cs[q][g]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int m = mb - q;
        if (full || m >= 0) {
            const float4 h = CORR ? __ldg(a.Hx + x0 + m) : f4(0.f, 0.f, 0.f, 0.f);
            float num = 0.f, den = 0.f;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float fin[4] = {fo[q][g].x, fo[q][g].y, fo[q][g].z, fo[q][g].w};
                float y[4];
#pragma unroll
                for (int p = 0; p < 4; ++p)
                    y[p] = cstep(p2_fwd<CORR>(fin[p], h, S[g][p]), p1[g][p], p2[g][p], q1[g][p], q2[g][p], k);
                if (OUT) {
                    num = fmaf(c.wt[g], fmaf(cs[q][g], y[2], sn[q][g] * y[3]), num);
                    den = fmaf(c.wt[g], fmaf(cs[q][g], y[0], sn[q][g] * y[1]), den);
                }
            }
            if (OUT && SM) {
                sb[m * 32] = make_float2(num, den);  // block-level group sum follows
            } else if (OUT && iv) {
                const size_t off = (size_t)(x0 + m) * FL_RB;
                pn[off] = num;
                pd[off] = den;
            }
        }
    }
}

template <int G>
__device__ __forceinline__ void p2_load_s0(const P2Ctx<G>& c, float (&S)[G][4][4]) {
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const float4 v = c.s0[g][p];
            S[g][p][0] = v.x;
            S[g][p][1] = v.y;
            S[g][p][2] = v.z;
            S[g][p][3] = v.w;
        }
}

template <int G, bool OUT, bool CORR, bool SM = false>
__device__ __forceinline__ void p2_tile_impl(const Pass2Args& a, const P2Ctx<G>& c, int t,
                                             float (&p1)[G][4], float (&p2)[G][4], float (&q1)[G][4],
                                             float (&q2)[G][4], float* pn, float* pd, bool iv,
                                             float2* sb) {
    const int x0 = t * TILE;
    const int len = min(TILE, a.W - x0);
    float S[G][4][4];
    if (CORR) p2_load_s0<G>(c, S);
    float4 fa[4][G], fb[4][G];
    float va[4], vb[4];
    if (len == TILE) {
        // 4 iterations of 8 steps: the recurrence state returns to the same
        // registers every iteration (no shuffling moves)
        p2_load4<G, OUT>(c, x0, TILE - 1, fa, va);
#pragma unroll 1
        for (int mb = TILE - 1; mb >= 7; mb -= 8) {
            p2_load4<G, OUT>(c, x0, mb - 4, fb, vb);
            p2_step4<G, OUT, CORR, SM>(a, c, x0, mb, true, fa, va, S, p1, p2, q1, q2, pn, pd, iv, sb);
            p2_load4<G, OUT>(c, x0, mb - 8, fa, va);  // clamped at x0 on the last iteration
            p2_step4<G, OUT, CORR, SM>(a, c, x0, mb - 4, true, fb, vb, S, p1, p2, q1, q2, pn, pd, iv, sb);
        }
    } else {
#pragma unroll 1
        for (int mb = len - 1; mb >= 0; mb -= 4) {
            p2_load4<G, OUT>(c, x0, mb, fa, va);
            p2_step4<G, OUT, CORR, SM>(a, c, x0, mb, false, fa, va, S, p1, p2, q1, q2, pn, pd, iv, sb);
        }
    }
}

// One tile right to left; the tiles left of nHx take the S0 correction.
template <int G, bool OUT, bool SM = false>
__device__ __forceinline__ void p2_tile(const Pass2Args& a, const P2Ctx<G>& c, int t,
                                        float (&p1)[G][4], float (&p2)[G][4], float (&q1)[G][4],
                                        float (&q2)[G][4], float* pn, float* pd, bool iv,
                                        float2* sb = nullptr) {
    if (t * TILE < a.nHx)
        p2_tile_impl<G, OUT, true, SM>(a, c, t, p1, p2, q1, q2, pn, pd, iv, sb);
    else
        p2_tile_impl<G, OUT, false, SM>(a, c, t, p1, p2, q1, q2, pn, pd, iv, sb);
}

// Exact forward output of one term at x (warm-up start of an x-chunk).
template <int G>
__device__ __forceinline__ void p2_fwd_at(const Pass2Args& a, const P2Ctx<G>& c, int g, int x,
                                          float (&F)[4]) {
    const float4 v = c.fl[g][(size_t)x * FL_RB];
    F[0] = v.x;
    F[1] = v.y;
    F[2] = v.z;
    F[3] = v.w;
    if (x < a.nHx) {
        const float4 h = __ldg(a.Hx + x);
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const float4 s = c.s0[g][p];
            F[p] = fmaf(h.x, s.x, fmaf(h.y, s.y, fmaf(h.z, s.z, fmaf(h.w, s.w, F[p]))));
        }
    }
}

// ---------------------------------------------------------------------------
// Pass 2 with the term groups of a block summed on chip: 4 warps = 32 rows x
// 4 groups of G terms (warp w = group 4*blockIdx.y + w).  Each warp stages
// its tile's (num, den) in shared memory; after a barrier the block adds the
// 4 groups in fixed order (deterministic) and writes one partial pair, so
// partial traffic (pass-2 writes + reduce reads) drops 4x.
constexpr int P2R_GR = 4;

#ifndef TBF_P2_NBUF
#define TBF_P2_NBUF 2  // staging buffers of the block-summed pass 2 (1: + a barrier per tile, half the smem)
#endif
#ifndef TBF_P2_MINB
#define TBF_P2_MINB 3  // k_pass2_gr blocks per SM requested from ptxas
#endif
constexpr int P2R_SMEM = TBF_P2_NBUF * P2R_GR * TILE * 32 * 8;  // float2 [NBUF][warp][x][row]

// LPT: unequal x-chunks (xlpt/xb1/xb2, dispatch order 4)
template <int G, bool LPT>
__global__ void __launch_bounds__(32 * P2R_GR, TBF_P2_MINB) k_pass2_gr(const __grid_constant__ Pass2Args a) {
    extern __shared__ float2 sdyn[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nsb = a.nrb_run * (P2_THREADS / 32);  // 32-row sub-blocks in this launch
    const int nch = gridDim.x / nsb;
    int chunk, rsb;
    int gy = blockIdx.y;  // group block
    if (LPT) {  // 1-D grid, chunk slowest (in xord order), then group block, row sub-block
        const int npb = (a.ngroups + P2R_GR - 1) / P2R_GR;
        int idx = blockIdx.x;
        rsb = idx % nsb;
        idx /= nsb;
        gy = idx % npb;
        chunk = (a.xord >> (2 * (idx / npb))) & 3;
    } else if (a.order == 1) {  // x-chunk fastest: both chunks of a row block together
        chunk = blockIdx.x % nch;
        rsb = blockIdx.x / nch;
    } else if (a.order == 2) {  // rows reversed within a chunk
        chunk = blockIdx.x / nsb;
        rsb = nsb - 1 - blockIdx.x % nsb;
    } else if (a.order == 3) {  // chunks reversed (rightmost, exact-start chunk first)
        chunk = nch - 1 - blockIdx.x / nsb;
        rsb = blockIdx.x % nsb;
    } else {
        chunk = blockIdx.x / nsb;
        rsb = blockIdx.x % nsb;
    }
    const int r0 = a.rb0 * P2_THREADS + rsb * 32;
    const int H = a.H, W = a.W;
    if (r0 >= H) return;  // whole block
    const int i_raw = r0 + lane;
    const bool iv = i_raw < H;
    const int i = iv ? i_raw : H - 1;
    const int grp_raw = gy * P2R_GR + w;
    const bool active = grp_raw < a.ngroups;
    const int grp = active ? grp_raw : a.ngroups - 1;
    const int b = blockIdx.z;
    // terms [term0, t.n) of the batch (term0 = 1 when the zero unit has its
    // own pass 2)
    const int j0 = a.term0 + grp * G;
    const int nt = min(G, a.t.n - j0);
    P2Ctx<G> c;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int j = min(j0 + g, a.t.n - 1);
        c.nu_hi[g] = a.t.nu_hi[j];
        c.nu_lo[g] = a.t.nu_lo[j];
        c.wt[g] = g < nt ? a.t.w[j] * a.wscale : 0.f;
        c.fl[g] = reinterpret_cast<const float4*>(a.floc) +
                  (((size_t)j * a.B + b) * ((H + FL_RB - 1) / FL_RB) + i / FL_RB) * W * (size_t)FL_RB + (i % FL_RB);
        c.s0[g] = reinterpret_cast<const float4*>(a.s0) + (((size_t)j * a.B + b) * H + i) * 4;
    }
    c.fT = a.fT + xm_index(b, 0, i, W, H);
    const size_t xpl = xm_plane(a.B, W, H);
    float* pn = a.part + (size_t)(gy * 2 + 0) * xpl + xm_index(b, 0, iv ? i_raw : 0, W, H);
    float* pd = a.part + (size_t)(gy * 2 + 1) * xpl + xm_index(b, 0, iv ? i_raw : 0, W, H);
    // tile k of this block stages in buffer k & 1: one barrier per tile (the
    // buffer written next was last read before the previous barrier)
    auto sbuf = [&](int buf, int q, int m) -> float2& { return sdyn[((buf * P2R_GR + q) * TILE + m) * 32 + lane]; };

    int t_lo, t_hi;  // exclusive
    if (LPT) {
        t_lo = chunk == 0 ? 0 : (chunk == 1 ? a.xb1 : a.xb2);
        t_hi = chunk == 0 ? a.xb1 : (chunk == 1 ? a.xb2 : a.ntx);
    } else {
        t_lo = chunk * a.tiles_per_chunk;
        t_hi = min(a.ntx, t_lo + a.tiles_per_chunk);
    }
    float p1[G][4], p2[G][4], q1[G][4], q2[G][4];
    if (active) {
        const bool exact_start = t_hi + a.warm_tiles >= a.ntx;
        if (exact_start) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int j = min(j0 + g, a.t.n - 1);
                const float4* bs = reinterpret_cast<const float4*>(a.bstate) + (((size_t)j * a.B + b) * H + i) * 4;
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const float4 v = bs[p];
                    p1[g][p] = v.x;
                    p2[g][p] = v.y;
                    q1[g][p] = v.z;
                    q2[g][p] = v.w;
                }
            }
#pragma unroll 1
            for (int t = a.ntx - 1; t >= t_hi; --t) p2_tile<G, false>(a, c, t, p1, p2, q1, q2, pn, pd, iv);
        } else {
            // warm-up: steady state of the exact forward output at the
            // warm-up start, then backward (no output) down to t_hi
            const int tw = min(a.ntx - 1, t_hi - 1 + a.warm_tiles);
            const int xs = min(W - 1, tw * TILE + TILE - 1);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                float F[4];
                p2_fwd_at<G>(a, c, g, xs, F);
#pragma unroll
                for (int p = 0; p < 4; ++p) csteady(F[p], p1[g][p], p2[g][p], q1[g][p], q2[g][p], a.k);
            }
#pragma unroll 1
            for (int t = tw; t >= t_hi; --t) p2_tile<G, false>(a, c, t, p1, p2, q1, q2, pn, pd, iv);
        }
    } else {
#pragma unroll
        for (int m = 0; m < TILE; ++m) {
            sbuf(0, w, m) = make_float2(0.f, 0.f);
            if (TBF_P2_NBUF > 1) sbuf(1, w, m) = make_float2(0.f, 0.f);
        }
    }
#pragma unroll 1
    for (int t = t_hi - 1, buf = 0; t >= t_lo; --t, buf = (buf + 1) % TBF_P2_NBUF) {
        if (active) p2_tile<G, true, true>(a, c, t, p1, p2, q1, q2, pn, pd, iv, &sbuf(buf, w, 0));
        __syncthreads();
        const int x0 = t * TILE;
        const int len = min(TILE, W - x0);
        if (iv) {
            for (int m = w; m < len; m += P2R_GR) {
                float2 acc = sbuf(buf, 0, m);
#pragma unroll
                for (int q = 1; q < P2R_GR; ++q) {
                    const float2 v = sbuf(buf, q, m);
                    acc.x += v.x;
                    acc.y += v.y;
                }
                const size_t off = (size_t)(x0 + m) * FL_RB;
                pn[off] = acc.x;
                pd[off] = acc.y;
            }
        }
        if (TBF_P2_NBUF == 1) __syncthreads();  // reads done before the next tile's stores
    }
}

// Zero unit, pass 2: thread = virtual row v (planes p = image rows v + p*hq),
// tiles right to left from the exact backward start (rightmost chunk) or a
// warm-up; F + Hx . S0 near x = 0 as in k_pass2_gr; no phasors (nu = 0).
__global__ void __launch_bounds__(128) k_pass2_zero(const __grid_constant__ ZeroArgs a) {
    const int v = blockIdx.x * 128 + threadIdx.x;
    if (v >= a.hq) return;
    const int chunk = blockIdx.y, b = blockIdx.z;
    const int H = a.H, W = a.W;
    const Casc k = a.k;
    const int nrbk = (H + FL_RB - 1) / FL_RB;
    const float4* fl = reinterpret_cast<const float4*>(a.floc) +
                       (((size_t)a.term * a.B + b) * nrbk + v / FL_RB) * W * (size_t)FL_RB + (v % FL_RB);
    const float4* s0 = reinterpret_cast<const float4*>(a.s0) + (((size_t)a.term * a.B + b) * H + v) * 4;
    auto fwd = [&](int x, float (&F)[4]) {
        const float4 t = ld_stream(fl + (size_t)x * FL_RB);
        F[0] = t.x;
        F[1] = t.y;
        F[2] = t.z;
        F[3] = t.w;
        if (x < a.nHx) {
            const float4 h = __ldg(a.Hx + x);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const float4 c = s0[p];
                F[p] = fmaf(h.x, c.x, fmaf(h.y, c.y, fmaf(h.z, c.z, fmaf(h.w, c.w, F[p]))));
            }
        }
    };
    const int t_lo = chunk * a.tiles_per_chunk;
    const int t_hi = min(a.ntx, t_lo + a.tiles_per_chunk);
    float p1[4], p2[4], q1[4], q2[4];
    int xs;
    if (t_hi + a.warm_tiles >= a.ntx) {  // exact start at the right edge
        const float4* bs = reinterpret_cast<const float4*>(a.bstate) + (((size_t)a.term * a.B + b) * H + v) * 4;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const float4 c = bs[p];
            p1[p] = c.x;
            p2[p] = c.y;
            q1[p] = c.z;
            q2[p] = c.w;
        }
        xs = W - 1;
    } else {  // warm-up from the steady state of the forward output
        xs = min(W - 1, (t_hi + a.warm_tiles) * TILE - 1);
        float F[4];
        fwd(xs, F);
#pragma unroll
        for (int p = 0; p < 4; ++p) csteady(F[p], p1[p], p2[p], q1[p], q2[p], k);
    }
    const int xo = min(W, t_hi * TILE);  // outputs for x < xo
    const int xlo = t_lo * TILE;
    // 4-step blocks, the next block's loads in flight meanwhile
    float4 cur[4], nxt[4];
    auto load4 = [&](int xb, float4 (&d)[4]) {
#pragma unroll
        for (int q = 0; q < 4; ++q) d[q] = ld_stream(fl + (size_t)max(xb - q, xlo) * FL_RB);
    };
    load4(xs, cur);
#pragma unroll 1
    for (int xb = xs; xb >= xlo; xb -= 4) {
        load4(xb - 4, nxt);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int x = xb - q;
            if (x < xlo) break;
            float F[4] = {cur[q].x, cur[q].y, cur[q].z, cur[q].w};
            if (x < a.nHx) {
                const float4 h = __ldg(a.Hx + x);
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const float4 c = s0[p];
                    F[p] = fmaf(h.x, c.x, fmaf(h.y, c.y, fmaf(h.z, c.z, fmaf(h.w, c.w, F[p]))));
                }
            }
            float y[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) y[p] = cstep(F[p], p1[p], p2[p], q1[p], q2[p], k);
            if (x < xo) {
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const int r = v + p * a.hq;
                    if (r < H) a.num[xm_index(b, x, r, W, H)] = a.wt * y[p];
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
    }
}

// ---------------------------------------------------------------------------
// Box variant (spatial.py:157-160, box_pass _core.pyx:28-53).  Pass 1 runs the
// normalised (2r+1) window along y as a running sum per column (fp64 sums;
// the reference keeps long double), modulation fused, and writes the
// y-filtered planes x-major through the smem transpose (same float4 tiled
// layout as F_loc).  Pass 2 runs the window along x per row, fused with
// demodulation.  Mirror indices follow _mirror (any radius, repeated
// reflection).  The box is FIR, so x-chunks of pass 2 are independent.
// ---------------------------------------------------------------------------

__device__ __forceinline__ float4 modulate4(float fv, float nu_hi, float nu_lo) {
    float s0, c0;
    sincos_fma(phase(nu_hi, nu_lo, fv), &s0, &c0);
    return make_float4(c0, s0, fv * c0, fv * s0);
}

template <int G, int R>
__global__ void __launch_bounds__(P1_WARPS * 32) k_pass1_box(const __grid_constant__ Pass1Args a, int radius) {
    extern __shared__ float smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int term = blockIdx.y * P1_WARPS + warp;
    if (term >= a.t.n) return;
    const int b = blockIdx.z;
    const int H = a.H, W = a.W;
    const int x0 = blockIdx.x * TILE;
    const int x = x0 + lane;
    const int xc = x < W ? x : W - 1;
    const int tlen = min(TILE, W - x0);
    float4* const buf = reinterpret_cast<float4*>(smem) + (size_t)warp * TILE * BUF_LD;
    float4* const bl = buf + lane;
    float4* const br = buf + lane * BUF_LD;
    const float nu_hi = a.t.nu_hi[term], nu_lo = a.t.nu_lo[term];
    const float* fcol = a.f + (size_t)b * H * W + xc;
    auto fy = [&](long long i) { return __ldg(fcol + (size_t)mirror_any(i, H) * W); };
    const double inv = 1.0 / (double)(2 * radius + 1);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (long long kk = -radius; kk <= radius; ++kk) {
        const float4 u = modulate4(fy(kk), nu_hi, nu_lo);
        acc[0] += u.x;
        acc[1] += u.y;
        acc[2] += u.z;
        acc[3] += u.w;
    }
    const int nrbk = (H + FL_RB - 1) / FL_RB;
    float4* const fl0 = reinterpret_cast<float4*>(a.floc) + ((size_t)term * a.B + b) * nrbk * W * (size_t)FL_RB;
    for (int i0 = 0; i0 < H; i0 += TILE) {
        const int len = min(TILE, H - i0);
        for (int r = 0; r < len; ++r) {
            const int i = i0 + r;
            bl[r * BUF_LD] = make_float4((float)(acc[0] * inv), (float)(acc[1] * inv),
                                         (float)(acc[2] * inv), (float)(acc[3] * inv));
            if (radius > 0 && i + 1 < H) {  // slide the window to row i+1
                const float4 un = modulate4(fy((long long)i + radius + 1), nu_hi, nu_lo);
                const float4 uo = modulate4(fy((long long)i - radius), nu_hi, nu_lo);
                acc[0] += (double)un.x - (double)uo.x;
                acc[1] += (double)un.y - (double)uo.y;
                acc[2] += (double)un.z - (double)uo.z;
                acc[3] += (double)un.w - (double)uo.w;
            } else if (radius == 0 && i + 1 < H) {
                const float4 u = modulate4(fy(i + 1), nu_hi, nu_lo);
                acc[0] = u.x;
                acc[1] = u.y;
                acc[2] = u.z;
                acc[3] = u.w;
            }
        }
        __syncwarp();
        const int i = i0 + lane;
        if (lane < len) {
            float4* fl = fl0 + ((size_t)(i / FL_RB) * W + x0) * FL_RB + (i % FL_RB);
            for (int xx = 0; xx < tlen; ++xx) fl[(size_t)xx * FL_RB] = br[xx];
        }
        __syncwarp();
    }
}

template <int G, int R>
__global__ void __launch_bounds__(P2_THREADS) k_pass2_box(const __grid_constant__ Pass2Args a, int radius) {
    const int chunk = blockIdx.x / a.nrb_run;
    const int i_raw = (a.rb0 + blockIdx.x % a.nrb_run) * P2_THREADS + threadIdx.x;
    const int H = a.H, W = a.W;
    const bool iv = i_raw < H;
    const int i = iv ? i_raw : H - 1;
    const int grp = blockIdx.y;
    const int b = blockIdx.z;
    const int j0 = grp * G;
    const int nt = min(G, a.t.n - j0);
    float nu_hi[G], nu_lo[G], wt[G];
    const float4* fl[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int j = min(j0 + g, a.t.n - 1);
        nu_hi[g] = a.t.nu_hi[j];
        nu_lo[g] = a.t.nu_lo[j];
        wt[g] = g < nt ? a.t.w[j] : 0.f;
        fl[g] = reinterpret_cast<const float4*>(a.floc) +
                (((size_t)j * a.B + b) * ((H + FL_RB - 1) / FL_RB) + i / FL_RB) * W * (size_t)FL_RB + (i % FL_RB);
    }
    const float* fT = a.fT + xm_index(b, 0, i, W, H);
    const size_t xpl = xm_plane(a.B, W, H);
    float* pn = a.part + (size_t)(grp * 2 + 0) * xpl + xm_index(b, 0, i_raw, W, H);
    float* pd = a.part + (size_t)(grp * 2 + 1) * xpl + xm_index(b, 0, i_raw, W, H);
    const int xa = chunk * a.tiles_per_chunk * TILE;
    const int xb = min(W, xa + a.tiles_per_chunk * TILE);
    const double inv = 1.0 / (double)(2 * radius + 1);
    auto Yx = [&](int g, long long xx) { return fl[g][(size_t)mirror_any(xx, W) * FL_RB]; };
    double acc[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.0;
        for (long long kk = (long long)xa - radius; kk <= (long long)xa + radius; ++kk) {
            const float4 v = Yx(g, kk);
            acc[g][0] += v.x;
            acc[g][1] += v.y;
            acc[g][2] += v.z;
            acc[g][3] += v.w;
        }
    }
    for (int xx = xa; xx < xb; ++xx) {
        float cc[G], sn[G];
        phasors<G, R>(fT[(size_t)xx * FL_RB], nu_hi, nu_lo, a.t.dnu, cc, sn);
        float num = 0.f, den = 0.f;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float y0 = (float)(acc[g][0] * inv), y1 = (float)(acc[g][1] * inv);
            const float y2 = (float)(acc[g][2] * inv), y3 = (float)(acc[g][3] * inv);
            num = fmaf(wt[g], fmaf(cc[g], y2, sn[g] * y3), num);
            den = fmaf(wt[g], fmaf(cc[g], y0, sn[g] * y1), den);
            if (xx + 1 < xb) {
                const float4 vn = Yx(g, (long long)xx + radius + 1);
                const float4 vo = Yx(g, (long long)xx - radius);
                if (radius > 0) {
                    acc[g][0] += (double)vn.x - (double)vo.x;
                    acc[g][1] += (double)vn.y - (double)vo.y;
                    acc[g][2] += (double)vn.z - (double)vo.z;
                    acc[g][3] += (double)vn.w - (double)vo.w;
                } else {
                    acc[g][0] = vn.x;
                    acc[g][1] = vn.y;
                    acc[g][2] = vn.z;
                    acc[g][3] = vn.w;
                }
            }
        }
        if (iv) {
            pn[(size_t)xx * FL_RB] = num;
            pd[(size_t)xx * FL_RB] = den;
        }
    }
}

// ---------------------------------------------------------------------------
// Reduce partial groups, transpose to row-major, optional guarded ratio.
// ---------------------------------------------------------------------------

// Tile of 32 x-rows by 128 rows (i): partials are read as float4 along i
// (512 B contiguous per warp and group), summed over groups in fixed order
// (deterministic), staged in smem, and written transposed (row-major).
constexpr int RED_I = 128;

__global__ void __launch_bounds__(256) k_reduce(const __grid_constant__ ReduceArgs a) {
    __shared__ float tn[TILE][RED_I + 4];
    __shared__ float td[TILE][RED_I + 4];
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * TILE, i0 = a.i_base + blockIdx.y * RED_I;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;  // 8 warps
    const size_t plane = xm_plane(a.B, a.W, a.H);
    const bool vec = true;  // row-block tiled partials: 4-row groups always aligned and padded
    for (int r = warp; r < TILE; r += 8) {
        const int gx = x0 + r;
        const int gi = i0 + 4 * lane;
        float n[4] = {0.f, 0.f, 0.f, 0.f}, d[4] = {0.f, 0.f, 0.f, 0.f};
        if (gx < a.W && gi < a.H) {
            const float* pp = a.part + xm_index(b, gx, gi, a.W, a.H);
            if (vec) {
                // up to 4 groups (8 float4 loads) in flight, also for a partial
                // block of groups (config 5 has 3 per batch), summed in fixed
                // group order
                for (int g = 0; g < a.ngroups; g += 4) {
                    float4 vn[4], vd[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (g + q < a.ngroups) {
                            vn[q] = __ldcs(reinterpret_cast<const float4*>(pp + (size_t)(2 * (g + q)) * plane));
                            vd[q] = __ldcs(reinterpret_cast<const float4*>(pp + (size_t)(2 * (g + q) + 1) * plane));
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (g + q < a.ngroups) {
                            n[0] += vn[q].x; n[1] += vn[q].y; n[2] += vn[q].z; n[3] += vn[q].w;
                            d[0] += vd[q].x; d[1] += vd[q].y; d[2] += vd[q].z; d[3] += vd[q].w;
                        }
                    }
                }
                if (a.zpart) {  // the zero unit last (fixed order)
                    const float4 vn = *reinterpret_cast<const float4*>(a.zpart + xm_index(b, gx, gi, a.W, a.H));
                    n[0] += vn.x; n[1] += vn.y; n[2] += vn.z; n[3] += vn.w;
                    d[0] += a.den_add; d[1] += a.den_add; d[2] += a.den_add; d[3] += a.den_add;
                }
            } else {
                const int cnt = min(4, a.H - gi);
                for (int g = 0; g < a.ngroups; ++g)
                    for (int q = 0; q < cnt; ++q) {
                        n[q] += pp[(size_t)(2 * g) * plane + q];
                        d[q] += pp[(size_t)(2 * g + 1) * plane + q];
                    }
                for (int q = 0; a.zpart && q < cnt; ++q) {
                    n[q] += a.zpart[xm_index(b, gx, gi, a.W, a.H) + q];
                    d[q] += a.den_add;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            tn[r][4 * lane + q] = n[q];
            td[r][4 * lane + q] = d[q];
        }
    }
    __syncthreads();
    unsigned long long guarded = 0;
    for (int rr = warp; rr < RED_I; rr += 8) {
        const int gi = i0 + rr, gx = x0 + lane;
        if (gi < a.H && gx < a.W) {
            const size_t off = ((size_t)b * a.H + gi) * a.W + gx;
            float n = tn[lane][rr], d = td[lane][rr];
            if (a.in_num) {
                n += a.in_num[off];
                d += a.in_den[off];
            }
            if (a.num) {
                a.num[off] = n;
                a.den[off] = d;
            }
            if (a.out) {
                const bool gd = !(d >= 1e-12f);
                guarded += gd;
                a.out[off] = gd ? a.f[off] : n / d;
            }
        }
    }
    if (a.out && a.counters) {
        // warp-aggregate then one atomic per warp (integer -> deterministic total)
        for (int o = 16; o > 0; o >>= 1) guarded += __shfl_down_sync(0xffffffffu, guarded, o);
        if (lane == 0 && guarded) atomicAdd(&a.counters[1], guarded);
    }
}

// Guarded ratio over n samples (engines.py:109-117), 4 samples per thread
// per step when the buffers are 16-byte aligned (the term-sharded root: 16
// B/px of streaming, ~0.7 ms at 16384^2), the same test per sample as k_reduce.
__global__ void k_finalize(const float* num, const float* den, const float* f, float* out,
                           long long n, unsigned long long* counters) {
    unsigned long long guarded = 0;
    auto one = [&](float nv, float d, float fv) {
        const bool gd = !(d >= 1e-12f);
        guarded += gd;
        return gd ? fv : nv / d;
    };
    const long long stride = (long long)gridDim.x * blockDim.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(num) | reinterpret_cast<uintptr_t>(den) |
                       reinterpret_cast<uintptr_t>(f) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    long long done = 0;
    if (vec) {
        const long long n4 = n / 4;
        for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n4; q += stride) {
            const float4 a = __ldcs(reinterpret_cast<const float4*>(num) + q);
            const float4 d = __ldcs(reinterpret_cast<const float4*>(den) + q);
            const float4 fv = __ldg(reinterpret_cast<const float4*>(f) + q);
            __stcs(reinterpret_cast<float4*>(out) + q,
                   make_float4(one(a.x, d.x, fv.x), one(a.y, d.y, fv.y), one(a.z, d.z, fv.z), one(a.w, d.w, fv.w)));
        }
        done = n4 * 4;
    }
    for (long long idx = done + blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n; idx += stride)
        out[idx] = one(num[idx], den[idx], f[idx]);
    for (int o = 16; o > 0; o >>= 1) guarded += __shfl_down_sync(0xffffffffu, guarded, o);
    if ((threadIdx.x & 31) == 0 && guarded && counters) atomicAdd(&counters[1], guarded);
}

__global__ void k_range_check(const float* f, long long n, double lo, double hi,
                              unsigned long long* counters) {
    unsigned long long bad = 0;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        double v = (double)f[idx];
        bad += !(v >= lo && v <= hi);  // NaN counts as bad
    }
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_down_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&counters[0], bad);
}

// f[b][i][x] -> fT[b][x][i]; with counters, also the range check of
// engines.py:218-225 on the same loads (counters[0] += samples outside
// [lo, hi] or NaN, as k_range_check)
__global__ void __launch_bounds__(256) k_transpose(const float* f, float* fT, float* fY, int H, int W,
                                                   double lo, double hi, unsigned long long* counters,
                                                   int tx0) {
    __shared__ float t[TILE][TILE + 1];
    const int b = blockIdx.z;
    const int x0 = (tx0 + blockIdx.x) * TILE, i0 = blockIdx.y * TILE;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const float* src = f + (size_t)b * H * W;
    float* const ytile = fY + ty_index(b, x0, i0, W, H);  // whole 32x32 tile (padding zeroed)
    unsigned bad = 0;
    for (int r = ty; r < TILE; r += 8) {
        int gi = i0 + r, gx = x0 + tx;
        const bool in = gi < H && gx < W;
        const float v = in ? src[(size_t)gi * W + gx] : 0.f;
        const double dv = (double)v;
        bad += in && !(dv >= lo && dv <= hi);
        t[r][tx] = v;
        ytile[r * 32 + tx] = v;
    }
    if (counters) {
        bad = __reduce_add_sync(0xffffffffu, bad);
        if (tx == 0 && bad) atomicAdd(&counters[0], (unsigned long long)bad);
    }
    __syncthreads();
    for (int r = ty; r < TILE; r += 8) {
        int gx = x0 + r, gi = i0 + tx;
        if (gx < W && gi < H) fT[xm_index(b, gx, gi, W, H)] = t[tx][r];
    }
}

// ---------------------------------------------------------------------------
// Plugin-level fp64 twins of _core.recursive_smooth / _core.box_pass.
// ---------------------------------------------------------------------------

__global__ void k_recursive_smooth_f64(const double* a, double* out, int h, int w, double scale,
                                       double c1, double c2, double c3, double c4, int pad,
                                       double* s) {
    const int xcol = blockIdx.x * blockDim.x + threadIdx.x;
    if (xcol >= w) return;
    const long long ext = (long long)h + 2LL * pad;
    auto S = [&](long long r) -> double& { return s[r * w + xcol]; };
    const double a0 = a[mirror_any(-pad, h) * w + xcol];
    for (int r = 0; r < 4; ++r) S(r) = a0;
    // Left-to-right, separately rounded products and sums (no FMA contraction),
    // i.e. the reference's own evaluation order -> bit-identical results.
    auto dot5 = [&](double x0, double x1, double x2, double x3, double x4) {
        double t = __dmul_rn(scale, x0);
        t = __dadd_rn(t, __dmul_rn(c1, x1));
        t = __dadd_rn(t, __dmul_rn(c2, x2));
        t = __dadd_rn(t, __dmul_rn(c3, x3));
        return __dadd_rn(t, __dmul_rn(c4, x4));
    };
    for (long long r = 0; r < ext; ++r) {
        const long long src = mirror_any(r - pad, h);
        S(r + 4) = dot5(a[src * w + xcol], S(r + 3), S(r + 2), S(r + 1), S(r));
    }
    for (long long r = ext + 4; r < ext + 8; ++r) S(r) = S(ext + 3);
    for (long long r = ext - 1; r >= 0; --r)
        S(r + 4) = dot5(S(r + 4), S(r + 5), S(r + 6), S(r + 7), S(r + 8));
    for (int r = 0; r < h; ++r) out[(long long)r * w + xcol] = S(pad + r + 4);
}

// Brute-force bilateral filter (engines.py:120-151 bilateral_direct), fp64:
// out = sum_w w*nb / sum_w w over the (2r+1)^2 window with weights
// taps[dy] taps[dx] range(nb - center), np.pad(mode="reflect") borders
// (repeated whole-sample reflection = mirror_any) and the guarded ratio
// (engines.py:109-117).  One block per output pixel; the block reduction has
// a fixed shape, so results are deterministic.  range kind 0: Gaussian
// exp(-s^2/(2 sigma^2)) (kernels.py:174-182); 1: raised cosine cos(omega s)^N
// (= trig_eval, kernels.py:161-171).
constexpr int BF_THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(BF_THREADS) k_bilateral_direct(const T* f, int B, int H, int W,
                                                                const int32_t* samples, long long n,
                                                                const double* taps, int r, int kind,
                                                                double param, int degree, double* out,
                                                                unsigned long long* guarded) {
    __shared__ double sn[BF_THREADS], sd[BF_THREADS];
    for (long long s = blockIdx.x; s < n; s += gridDim.x) {
        int b, y, x;
        if (samples) {
            b = samples[3 * s];
            y = samples[3 * s + 1];
            x = samples[3 * s + 2];
        } else {
            b = (int)(s / ((long long)H * W));
            const long long rem = s - (long long)b * H * W;
            y = (int)(rem / W);
            x = (int)(rem - (long long)y * W);
        }
        const T* F = f + (size_t)b * H * W;
        const double c = (double)F[(size_t)y * W + x];
        const int win = 2 * r + 1;
        const long long taps2 = (long long)win * win;
        double num = 0.0, den = 0.0;
        const double inv2s2 = kind == 0 ? 1.0 / (2.0 * param * param) : 0.0;
        for (long long t = threadIdx.x; t < taps2; t += BF_THREADS) {
            const int dy = (int)(t / win) - r, dx = (int)(t % win) - r;
            const long long yy = mirror_any((long long)y + dy, H), xx = mirror_any((long long)x + dx, W);
            const double nb = (double)F[(size_t)yy * W + xx];
            const double d = nb - c;
            double rw;
            if (kind == 0) {
                rw = exp(-(d * d) * inv2s2);
            } else {
                double base = cos(param * d);
                rw = 1.0;
                for (int e = degree; e > 0; e >>= 1) {  // base^degree by squaring
                    if (e & 1) rw *= base;
                    base *= base;
                }
            }
            const double wgt = taps[dy + r] * taps[dx + r] * rw;
            num += wgt * nb;
            den += wgt;
        }
        sn[threadIdx.x] = num;
        sd[threadIdx.x] = den;
        __syncthreads();
        for (int o = BF_THREADS / 2; o > 0; o >>= 1) {
            if (threadIdx.x < o) {
                sn[threadIdx.x] += sn[threadIdx.x + o];
                sd[threadIdx.x] += sd[threadIdx.x + o];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const bool gd = sd[0] < 1e-12;
            out[s] = gd ? c : sn[0] / sd[0];
            if (gd && guarded) atomicAdd(guarded, 1ULL);
        }
        __syncthreads();
    }
}

__global__ void k_box_pass_f64(const double* a, double* out, int h, int w, int radius) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= h) return;
    const double* ar = a + (long long)row * w;
    double* orow = out + (long long)row * w;
    if (radius == 0) {
        for (int j = 0; j < w; ++j) orow[j] = ar[j];
        return;
    }
    // Kahan-compensated running sum (the reference keeps long double)
    double acc = 0.0, comp = 0.0;
    auto add = [&](double v) {
        double y = v - comp;
        double t = acc + y;
        comp = (t - acc) - y;
        acc = t;
    };
    for (long long k = -radius; k <= radius; ++k) add(ar[mirror_any(k, w)]);
    const double inv = 1.0 / (double)(2 * radius + 1);
    orow[0] = acc * inv;
    for (int j = 1; j < w; ++j) {
        add(ar[mirror_any((long long)j + radius, w)]);
        add(-ar[mirror_any((long long)j - radius - 1, w)]);
        orow[j] = acc * inv;
    }
}

// ---------------------------------------------------------------------------
// Host side: plan, workspace layout, launches.
// ---------------------------------------------------------------------------

constexpr int G1 = 1;  // terms per pass-1 warp == phasor anchor block R
constexpr int G2 = 2;  // terms per pass-2 thread (multiple of G1)
constexpr int R_ANCHOR = G1;
constexpr int TAB_PAD = 16;  // zero padding past the last term of the table
// term table [nu_hi | nu_lo | w] (ld = n + TAB_PAD each), then the float4
// right-extension coefficients bx at a 16-byte aligned offset (in floats)
inline size_t tab_bx_offset(int nterms) { return ((size_t)3 * (nterms + TAB_PAD) + 3) / 4 * 4; }

size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

struct Layout {
    int B, H, W, Ey, Ex, nseg, ntx, ne, edge_all;
    int row0, row1;  // output rows (a band for the term-sharded leftover terms, else [0, H))
    int zhq;         // zero unit: virtual rows (a quarter of H in whole 32-row segments)
    int nst;  // stripes of P1_WARPS column tiles (pass-1 blocks per term and y-chunk)
    int nyc, ych_rows, ywarm;  // pass-1 y-chunking (nseg = checkpoint segments per chunk)
    int ychb[TBF_MAX_YCH + 1];  // chunk boundaries (ych_rows = the largest chunk)
    bool ych_lpt;               // chunks of unequal size, dispatched largest first
    int tb;     // terms per batch (multiple of G2)
    int ng2;    // pass-2 groups per batch
    int nb;     // batches
    int nslot;  // batch buffer sets (2 = pass 1 of batch k+1 overlaps the rest of batch k)
    // shared buffers
    size_t off_fT, off_fY, off_num, off_den, off_tab;
    // per-slot buffers (offsets relative to the slot base)
    size_t off_slot, slot_bytes;
    size_t s_ckpt, s_floc, s_mail, s_flags, s_edge, s_s0, s_bst, s_part;
    size_t total;
};

int g_pass1_fold = 1;   // tbf_set_option(TBF_OPT_P1_FOLD); see run_terms
int g_p1_ychunks = 0;   // tbf_set_option(TBF_OPT_P1_YCHUNKS): 0 = automatic
int g_lpt_split = 3;    // tbf_set_option(TBF_OPT_LPT_SPLIT): bits 1/2 = planned unequal y-/x-chunks for few-wave launches,
                        // 4/8 = also in the host entry's strip/band launches
int g_p1_occ = 3;       // tbf_set_option(TBF_OPT_P1_OCC): pass-1 blocks per SM (2 leaves room for a pass-2 block)
int g_p2_chunks = 0;    // tbf_set_option(TBF_OPT_P2_CHUNKS): 0 = automatic
int g_pipeline = 0;     // tbf_set_option(TBF_OPT_PIPELINE) (measured: no gain on B200, SMs time-slice)
int g_auto_batches = 2; // tbf_set_option(TBF_OPT_BATCHES): batches when batch_terms <= 0
int g_p2_order = 0;     // tbf_set_option(TBF_OPT_P2_ORDER): block order of the block-summed pass 2 (same-box A/B: orders 0 and 1 equal)
int g_host_strips = 0;  // tbf_set_option(TBF_OPT_HOST_STRIPS): column strips of the host input (0 auto)
int g_host_bands = 0;   // tbf_set_option(TBF_OPT_HOST_BANDS): row bands of the host output (0 auto)
int g_p1_cluster = 1;   // tbf_set_option(TBF_OPT_P1_CLUSTER): stripes per pass-1 thread-block cluster
                        // (1 = none, the default: clusters of 4 measured 2-6% slower)
int g_zero_unit = 0;    // tbf_set_option(TBF_OPT_ZERO_UNIT): the zero frequency as a packed 1-plane unit
                        // (measured slower end to end: off by default)

// Pass-1 y-chunk planner for launches of a few waves.  Blocks of one chunk
// level all cost the same; the levels are dispatched largest first (block
// order with the chunk index slowest), and the makespan is that of list
// scheduling onto the resident block slots.  Block cost = instructions per
// row of the phases it runs: phase A (forward, ~24 per row), phase B
// (forward recompute + backward, ~43) and the epilogue (~18 per output row),
// from the ncu source page (profiles/ DESIGN.md 9).  Measured on config 2
// (B200): the simulated best split (1408 + 640 rows) was also the measured
// best, 6% less pass-1 time than two equal chunks (tail wave at partial
// occupancy).
double lpt_makespan(std::vector<double> d, long long per_level, int slots) {
    std::sort(d.begin(), d.end(), std::greater<double>());  // costliest level first
    std::priority_queue<double, std::vector<double>, std::greater<double>> q;
    for (int s = 0; s < slots; ++s) q.push(0.0);
    double mk = 0.0;
    for (double dl : d)
        for (long long j = 0; j < per_level; ++j) {
            const double t = q.top() + dl;
            q.pop();
            q.push(t);
            mk = std::max(mk, t);
        }
    return mk;
}

double p1_makespan(const std::vector<int>& bnd, int H, int Ey, int ywarm, long long per_chunk, int slots) {
    std::vector<double> d;
    for (size_t c = 0; c + 1 < bnd.size(); ++c) {
        const int R0 = bnd[c], R1 = bnd[c + 1];
        const int A0 = R0 - ywarm <= 0 ? -Ey : R0 - ywarm;
        const int Bend = R1 + ywarm >= H + Ey ? H + Ey : R1 + ywarm;
        d.push_back(24.0 * (Bend - A0) + 43.0 * (Bend - R0) + 18.0 * (R1 - R0));
    }
    return lpt_makespan(d, per_chunk, slots);
}

// Pass-2 x-chunk cost: tiles walked, including the warm-up tiles of every
// chunk but the rightmost (exact start).
double p2_chunk_cost(int t0, int t1, int ntx, int warm) {
    return (double)((t1 + warm >= ntx ? ntx : t1 + warm) - t0);
}

// Best split of the ntx column tiles of a pass-2 row into x-chunks (1..3,
// dispatched costliest first) by lpt_makespan, against the equal split of
// `uniform` chunks (kept on near ties).  Cached per shape.  Measured on config 2
// (B200): 48 + 16 tiles, costliest first, took 9% less pass-2 time than the
// 4 x 16 equal split; pass 2 streams HBM, so a tail wave at partial occupancy
// runs below bandwidth.
std::vector<int> p2_plan_split(int ntx, int warm, int uniform, long long per_chunk, int slots) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, long long, int>, std::vector<int>> cache;
    const auto key = std::make_tuple(ntx, warm, uniform, per_chunk, slots);
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    auto eval = [&](const std::vector<int>& b) {
        std::vector<double> d;
        for (size_t c = 0; c + 1 < b.size(); ++c) d.push_back(p2_chunk_cost(b[c], b[c + 1], ntx, warm));
        return lpt_makespan(d, per_chunk, slots);
    };
    const int tpc = (ntx + uniform - 1) / uniform;
    std::vector<int> best{0};
    for (int c = 1; c * tpc < ntx + tpc; ++c) best.push_back(std::min(ntx, c * tpc));
    best.back() = ntx;
    double best_mk = eval(best);
    auto consider = [&](std::vector<int> b) {
        const double mk = eval(b);
        if (mk < best_mk * 0.97) {
            best_mk = mk;
            best = b;
        }
    };
    for (int a = 1; a < ntx; ++a) consider({0, a, ntx});
    const int st = std::max(1, ntx / 32);
    for (int a = 1; a < ntx; a += st)
        for (int b2 = a + 1; b2 < ntx; b2 += st) consider({0, a, b2, ntx});
    std::lock_guard<std::mutex> g(mu);
    cache[key] = best;
    return best;
}

// Best split of H rows (multiples of TILE, each >= minr, non-increasing) into
// 1..3 chunks by p1_makespan; cached per shape.  Returns the boundaries.
std::vector<int> p1_plan_split(int H, int Ey, int ywarm, long long per_chunk, int slots) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, long long, int>, std::vector<int>> cache;
    const auto key = std::make_tuple(H, Ey, ywarm, per_chunk, slots);
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    const int units = (H + TILE - 1) / TILE;  // 32-row units (the last may be partial)
    const int minu = std::max(2, (ywarm + TILE - 1) / TILE);
    std::vector<int> best{0, H};
    double best_mk = p1_makespan(best, H, Ey, ywarm, per_chunk, slots);
    auto consider = [&](std::vector<int> u) {  // chunk sizes in units, largest first
        std::vector<int> b{0};
        for (size_t i = 0; i < u.size(); ++i) b.push_back(i + 1 == u.size() ? H : std::min(H, b.back() + u[i] * TILE));
        const double mk = p1_makespan(b, H, Ey, ywarm, per_chunk, slots);
        if (mk < best_mk * 0.99) {  // fewer chunks on near ties (candidates come in increasing count)
            best_mk = mk;
            best = b;
        }
    };
    for (int a = (units + 1) / 2; a <= units - minu; ++a) consider({a, units - a});
    const int step3 = std::max(1, units / 24);
    for (int a = (units + 2) / 3; a <= units - 2 * minu; a += step3)
        for (int b2 = minu; b2 <= std::min(a, units - a - minu); b2 += step3) {
            const int c = units - a - b2;
            if (c < minu || c > b2) continue;
            consider({a, b2, c});
        }
    std::lock_guard<std::mutex> g(mu);
    cache[key] = best;
    return best;
}

// lpt: 0 equal y-chunks (the host entry's strip-wise pass 1), 1 planned
// unequal chunks when TBF_OPT_LPT_SPLIT enables them, 2 planned regardless of
// the option (workspace sizing: a plan must fit whatever the option is later)
int make_layout(int B, int H, int W, const tbf_spatial* sp, int nterms_range, int batch_terms,
                Layout* L, int lpt = 1, int row0 = 0, int row1 = -1) {
    if (B < 1 || H < 1 || W < 1) return fail(TBF_ERR_DIM, "bad shape B=%d H=%d W=%d", B, H, W);
    if (!sp) return fail(TBF_ERR_PARAM, "null spatial");
    if (row1 < 0) row1 = H;
    // output rows [row0, row1): a band of whole 128-row pass-2 blocks (the
    // term-sharded path splits leftover terms by bands); planned chunks only
    // for the whole image
    if (row0 < 0 || row1 > H || row0 >= row1 || row0 % P2_THREADS || (row1 % P2_THREADS && row1 != H))
        return fail(TBF_ERR_PARAM, "bad row band [%d, %d) of %d (multiples of %d)", row0, row1, H, P2_THREADS);
    const bool band = row0 > 0 || row1 < H;
    if (band) lpt = 0;
    L->row0 = row0;
    L->row1 = row1;
    const int Hb = row1 - row0;
    L->B = B;
    L->H = H;
    L->W = W;
    const bool box = sp->kind == TBF_SPATIAL_BOX;
    L->Ey = box ? 0 : std::max(0, std::min(sp->ext_y, H - 1));
    L->Ex = box ? 0 : std::max(0, std::min(sp->ext_x, W - 1));
    L->ntx = (W + TILE - 1) / TILE;
    L->nst = (W + STRIPE - 1) / STRIPE;
    L->edge_all = 2 * (L->Ex + 1) >= W;
    L->ne = L->edge_all ? W : 2 * (L->Ex + 1);
    int tb;
    if (batch_terms > 0) {
        tb = std::min(batch_terms, nterms_range);
    } else {
        // automatic: a few batches so pass 1 of one batch overlaps the memory-
        // bound rest of the previous one (when pipelining is on)
        const int nbat = (g_pipeline && !box) ? std::max(1, g_auto_batches) : 1;
        tb = (nterms_range + nbat - 1) / nbat;
    }
    tb = std::max(tb, 1);
    tb = (tb + G2 - 1) / G2 * G2;  // whole groups, so anchors stay aligned across batches
    L->tb = tb;
    L->ng2 = tb / G2;
    L->nb = (nterms_range + tb - 1) / tb;
    L->nslot = (g_pipeline && !box && L->nb > 1) ? 2 : 1;
    // pass-1 y-chunking: split columns into chunks of rows (each with ywarm
    // warm-up rows on its inner sides) to fill the GPU.  Cost model fitted on
    // B200 sweeps (round 1, configs 1/2/4): a block's time is its row count;
    // above one wave of blocks the kernel takes (waves + 0.9) block times
    // (tail), below one wave a single block time.
    L->ywarm = (std::max(sp->ext_y, 1) + TILE - 1) / TILE * TILE;
    L->nyc = 1;
    L->ych_rows = H;
    if (!box) {
        const double slots = 148.0 * P1_BLOCKS_PER_SM;
        const double blocks1 = (double)L->nst * tb * B;
        double best = -1.0;
        int best_n = 1;
        for (int nyc = 1; nyc <= 16; ++nyc) {
            const int rows = ((Hb + nyc - 1) / nyc + TILE - 1) / TILE * TILE;
            const int n = (Hb + rows - 1) / rows;
            if (n != nyc) continue;  // same split as a smaller count
            // chunks shorter than the warm-up only while the launch stays
            // under one wave (long decays on small images: parallelism
            // matters more than the warm-up rows)
            if (nyc > 1 && rows < L->ywarm && blocks1 * nyc > slots) break;
            // rows the longest chunk sweeps: its output rows plus warm-ups,
            // clamped to the mirror extension [-Ey, H + Ey)
            double len = 0.0;
            for (int c = 0; c < n; ++c) {
                const int R0 = row0 + c * rows, R1 = std::min(row1, R0 + rows);
                const int A0 = (nyc == 1 && !band) ? -L->Ey : std::max(R0 - L->ywarm, -L->Ey);
                const int A1 = (nyc == 1 && !band) ? H + L->Ey : std::min(R1 + L->ywarm, H + L->Ey);
                len = std::max(len, (double)(A1 - A0));
            }
            const double waves = blocks1 * nyc / slots;
            const double cost = len * (waves <= 1.0 ? 1.0 : waves + 0.9);
            if (best < 0 || cost < best * 0.98) {  // prefer fewer chunks on near ties
                best = cost;
                best_n = nyc;
            }
        }
        int nyc = best_n;
        if (g_p1_ychunks > 0) {
            // forced count: at most TBF_MAX_YCH chunks (ychb[] bound), none
            // shorter than the warm-up (the automatic search's own limit)
            const int max_by_warm = std::max(1, Hb / std::max(L->ywarm, TILE));
            nyc = std::min(std::min(g_p1_ychunks, TBF_MAX_YCH), std::min((Hb + TILE - 1) / TILE, max_by_warm));
        }
        L->ych_rows = ((Hb + nyc - 1) / nyc + TILE - 1) / TILE * TILE;
        L->nyc = (Hb + L->ych_rows - 1) / L->ych_rows;
    }
    for (int c = 0; c <= L->nyc; ++c) L->ychb[c] = std::min(row1, row0 + c * L->ych_rows);
    L->ych_lpt = false;
    // single-batch runs only: the workspace of batched runs stays affine in
    // the batch size (the engine's batch picker fits it), and their launches
    // are many waves anyway (config 5)
    if (!box && g_p1_ychunks <= 0 && (lpt == 2 || (lpt == 1 && (g_lpt_split & 1))) && L->nb == 1) {
        // few waves: plan unequal chunks, largest first (p1_plan_split)
        const int slots = 148 * P1_BLOCKS_PER_SM;
        const long long per_chunk = (long long)L->nst * tb * B;
        // (not for short columns or launches under a wave per chunk level:
        // config 1, 512 rows and 64 blocks, was 6% slower with the planned
        // 3-way split; such launches are latency-bound, which the model does
        // not describe)
        if (per_chunk < 6LL * slots && per_chunk >= slots && H >= 1024 && H >= 16 * L->ywarm) {
            const std::vector<int> b = p1_plan_split(H, L->Ey, L->ywarm, per_chunk, slots);
            L->nyc = (int)b.size() - 1;
            L->ych_rows = 0;
            for (int c = 0; c < L->nyc; ++c) L->ych_rows = std::max(L->ych_rows, b[c + 1] - b[c]);
            for (int c = 0; c <= L->nyc; ++c) L->ychb[c] = b[c];
            L->ych_lpt = L->nyc > 1;
        }
    }
    if (!box && !band) {
        // development override: explicit chunk row counts, e.g. "1280,768"
        // (multiples of 32, largest first; the last one takes the rest)
        const char* ev = getenv("TBF_P1_YSPLIT");
        if (ev && *ev) {
            int n = 0, r = 0, mx = 0;
            L->ychb[0] = 0;
            for (const char* q = ev; *q && n < 3 && r < H;) {  // at most 3 chunks
                int v = (int)strtol(q, (char**)&q, 10);
                if (*q == ',') ++q;
                v = std::max(TILE, (v + TILE - 1) / TILE * TILE);
                if (!*q || n == 2) v = H - r;
                v = std::min(v, H - r);
                r += v;
                mx = std::max(mx, v);
                L->ychb[++n] = r;
            }
            if (r < H) {
                mx = std::max(mx, H - r);
                L->ychb[n] = H;
            }
            L->nyc = n;
            L->ych_rows = mx;
            L->ych_lpt = n > 1;
        }
    }
    // the zero unit's chunk: the virtual rows (row quarters) plus Ey both ways
    L->zhq = ((H + 3) / 4 + TILE - 1) / TILE * TILE;
    auto seg_count = [&]() {
        int ns = (L->ych_rows + std::max(L->ywarm, L->Ey) + TILE - 1) / TILE + 1;
        if (!box) ns = std::max(ns, (L->zhq + 2 * L->Ey + TILE - 1) / TILE + 1);
        return ns;
    };
    L->nseg = seg_count();
    if (band && !box) {
        // the workspace is sized for the whole image (tbf_workspace_bytes has no
        // band): a band's chunks may not need more checkpoint segments than the
        // whole image's equal chunks; fewer, longer chunks until they fit
        Layout F;
        if (make_layout(B, H, W, sp, nterms_range, batch_terms, &F, 0) == TBF_OK) {
            const long long cap = (long long)F.nyc * F.nseg;
            while (L->nyc > 1 && (long long)L->nyc * L->nseg > cap) {
                const int nyc = L->nyc - 1;
                L->ych_rows = ((Hb + nyc - 1) / nyc + TILE - 1) / TILE * TILE;
                L->nyc = (Hb + L->ych_rows - 1) / L->ych_rows;
                for (int c = 0; c <= L->nyc; ++c) L->ychb[c] = std::min(row1, row0 + c * L->ych_rows);
                L->nseg = seg_count();
            }
        }
    }
    const size_t px = (size_t)B * H * W;
    size_t o = 0;
    L->off_fT = o;
    o = align_up(o + xm_plane(B, W, H) * 4);
    L->off_fY = o;
    o = align_up(o + ty_plane(B, W, H) * 4);
    const bool multi = L->nb > 1;
    L->off_num = o;
    if (multi) o = align_up(o + px * 4);
    L->off_den = o;
    if (multi) o = align_up(o + px * 4);
    L->off_tab = o;
    o = align_up(o + (tab_bx_offset(nterms_range) + (size_t)4 * L->Ex + (size_t)4 * L->ntx * TILE) * 4);
    // one slot
    size_t q = 0;
    L->s_ckpt = q;
    if (!box) q = align_up(q + (size_t)L->nyc * L->nseg * tb * 16 * B * W * 4);
    L->s_floc = q;  // row-block tiled like xm_index (padded to whole FL_RB-row blocks)
    q = align_up(q + (size_t)tb * 4 * B * W * ((size_t)(H + FL_RB - 1) / FL_RB * FL_RB) * 4);
    L->s_mail = q;  // pass-1 x chain hand-off: float4 [tb][B][nst+1][H][4]
    if (!box) q = align_up(q + (size_t)tb * 16 * B * (L->nst + 1) * H * 4);
    L->s_flags = q;  // [tb][B][nst][ceil(H/32)] hand-off flags + the dispatch tickets
    if (!box) q = align_up(q + ((size_t)tb * B * L->nst * ((H + TILE - 1) / TILE) + P1_MAX_LAUNCHES) * 4);
    L->s_edge = q;
    if (!box) q = align_up(q + (size_t)tb * 4 * B * L->ne * H * 4);
    L->s_s0 = q;
    if (!box) q = align_up(q + (size_t)tb * 16 * B * H * 4);
    L->s_bst = q;
    if (!box) q = align_up(q + (size_t)tb * 16 * B * H * 4);
    // the (num, den) pairs of the pass-2 group blocks (box: one per G2-term
    // group; Gaussian: k_pass2_gr sums P2R_GR groups per block), then the zero
    // unit's num plane
    L->s_part = q;
    const size_t npairs = box ? (size_t)L->ng2 : (size_t)(L->ng2 + P2R_GR - 1) / P2R_GR;
    q = align_up(q + (npairs + 1) * 2 * xm_plane(B, W, H) * 4);
    L->slot_bytes = q;
    L->off_slot = o;
    o += (size_t)L->nslot * q;
    L->total = o;
    return TBF_OK;
}

// Internal streams per device: 0 = pipelined batches, 1 = host->device
// copies, 2/3 = pass-1 strips and pass-2 bands of the host pipeline, 4 =
// device->host copies, 5 = the zero unit's passes.
constexpr int N_AUX = 6;
cudaStream_t aux_stream(int idx = 0) {
    static std::mutex mu;
    static cudaStream_t streams[64][N_AUX] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (dev < 0 || dev >= 64 || idx < 0 || idx >= N_AUX) return nullptr;
    if (!streams[dev][idx]) cudaStreamCreateWithFlags(&streams[dev][idx], cudaStreamNonBlocking);
    return streams[dev][idx];
}

// Small pool of timing-free events (reused across calls).
cudaEvent_t event_get() {
    static std::mutex mu;
    static std::vector<cudaEvent_t> pool;
    static size_t next = 0;
    std::lock_guard<std::mutex> g(mu);
    if (pool.size() < 256) {
        cudaEvent_t e;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        pool.push_back(e);
        return e;
    }
    return pool[next++ % pool.size()];
}

// Response of the pure cascade to a unit state at x = 0 with zero input:
// hx[x] = output at sample x for each of the 4 unit states (what pass 2 adds
// to the zero-start chain, times the left-extension state S0), kept up to
// nHx = the whole tiles that cover every sample where it exceeds 1e-9 of its
// peak (at most W); MW = the state after all W samples (column-major, what
// the edge kernel adds to the chain's end state).  Double precision.
void left_response(const tbf_spatial* sp, int W, std::vector<float>& hx, int& nHx, double MW[16]) {
    std::vector<double> h((size_t)W * 4);
    double peak = 0.0;
    for (int kk = 0; kk < 4; ++kk) {
        double v1 = kk == 0, v2 = kk == 1, y1 = kk == 2, y2 = kk == 3;
        for (int x = 0; x < W; ++x) {
            const double v = sp->a1 * v1 + sp->a2 * v2;
            v2 = v1;
            v1 = v;
            const double y = v + sp->b1 * y1 + sp->b2 * y2;
            y2 = y1;
            y1 = y;
            h[(size_t)x * 4 + kk] = y;
            peak = std::max(peak, std::fabs(y));
        }
        MW[kk * 4 + 0] = v1;
        MW[kk * 4 + 1] = v2;
        MW[kk * 4 + 2] = y1;
        MW[kk * 4 + 3] = y2;
    }
    int last = 0;
    for (int x = 0; x < W; ++x)
        for (int kk = 0; kk < 4; ++kk)
            if (std::fabs(h[(size_t)x * 4 + kk]) > 1e-9 * peak) last = x + 1;
    nHx = std::min(W, (last + TILE - 1) / TILE * TILE);
    const int ntile = (nHx + TILE - 1) / TILE * TILE;
    hx.assign((size_t)ntile * 4, 0.f);
    for (int x = 0; x < std::min(ntile, W); ++x)
        for (int kk = 0; kk < 4; ++kk) hx[(size_t)x * 4 + kk] = (float)h[(size_t)x * 4 + kk];
}

// Closed form of the chain's right x-extension (spatial.py:171 mirror pad,
// _core.pyx:75-92): forward over Ex mirrored samples from the state s at
// x = W, steady start from the last output, backward over the Ex outputs.
// Linear in (s, inputs): bstate = Rx . s + sum_e bx[e] * Y(W-2-e), per plane.
// Evaluated in double with the kernels' pure-cascade steps; cached.
void right_ext_coeffs(const tbf_spatial* sp, int Ex, double Rx[16], std::vector<float>& bx) {
    static std::mutex mu;
    static double key[7] = {0, 0, 0, 0, 0, 0, -1};
    static double cR[16];
    static std::vector<float> cb;
    std::lock_guard<std::mutex> g(mu);
    const double kk[7] = {sp->a1, sp->a2, sp->b1, sp->b2, sp->g1, sp->g2, (double)Ex};
    if (std::equal(kk, kk + 7, key)) {
        std::copy(cR, cR + 16, Rx);
        bx = cb;
        return;
    }
    const double ig1 = 1.0 / sp->g1, ig = 1.0 / (sp->g1 * sp->g2);
    std::vector<double> outs(std::max(Ex, 1));
    bx.assign((size_t)Ex * 4, 0.f);
    for (int k = 0; k < 4 + Ex; ++k) {
        double v1 = k == 0, v2 = k == 1, y1 = k == 2, y2 = k == 3;
        double last = y1;
        for (int e = 0; e < Ex; ++e) {
            const double u = (k >= 4 && e == k - 4) ? 1.0 : 0.0;
            const double v = u + sp->a1 * v1 + sp->a2 * v2;
            v2 = v1;
            v1 = v;
            const double y = v + sp->b1 * y1 + sp->b2 * y2;
            y2 = y1;
            y1 = y;
            outs[e] = last = y;
        }
        double p1 = last * ig1, p2 = p1, q1 = last * ig, q2 = q1;
        for (int e = Ex - 1; e >= 0; --e) {
            const double v = outs[e] + sp->a1 * p1 + sp->a2 * p2;
            p2 = p1;
            p1 = v;
            const double y = v + sp->b1 * q1 + sp->b2 * q2;
            q2 = q1;
            q1 = y;
        }
        const double r[4] = {p1, p2, q1, q2};
        for (int c = 0; c < 4; ++c) {
            if (k < 4)
                Rx[k * 4 + c] = r[c];
            else
                bx[(size_t)(k - 4) * 4 + c] = (float)r[c];
        }
    }
    std::copy(kk, kk + 7, key);
    std::copy(Rx, Rx + 16, cR);
    cb = bx;
}

Casc to_casc(const tbf_spatial* sp) {
    const double g = sp->g1 * sp->g2;
    return Casc{(float)sp->a1, (float)sp->a2, (float)sp->b1, (float)sp->b2,
                (float)(1.0 / sp->g1), (float)(1.0 / g), (float)(g * g)};
}

int validate(const tbf_spatial* sp, const tbf_terms* terms, int tbeg, int tend) {
    if (!sp || !terms) return fail(TBF_ERR_PARAM, "null spatial/terms");
    if (sp->kind != TBF_SPATIAL_RECURSIVE && sp->kind != TBF_SPATIAL_BOX)
        return fail(TBF_ERR_PARAM, "unknown spatial kind %d", sp->kind);
    if (sp->kind == TBF_SPATIAL_BOX && sp->radius < 0)
        return fail(TBF_ERR_PARAM, "box radius must be >= 0, got %d", sp->radius);
    if (terms->n_terms < 1 || !terms->nu || !terms->weight)
        return fail(TBF_ERR_PARAM, "no terms");
    if (tbeg < 0 || tend > terms->n_terms || tbeg >= tend)
        return fail(TBF_ERR_PARAM, "bad term range [%d,%d) of %d", tbeg, tend, terms->n_terms);
    return TBF_OK;
}

constexpr int P1_SMEM = P1_WARPS * 4 * G1 * TILE * BUF_LD * 4;
// Gaussian pass 1: the segment tiles plus the x hand-off slots between the
// stripe's warps and the incoming slot of a cluster hand-off (75.8 KB: 3
// blocks per SM still fit the 228 KB)
constexpr int P1_SMEM_GAUSS = P1_SMEM + P1_WARPS * 4 * TILE * 16;  // + the incoming cluster slot: 75.8 KB
constexpr int P1_SMEM_OCC2 = 80 * 1024;  // padded request: at most 2 pass-1 blocks per SM

// cudaFuncSetAttribute applies to the current device only: done once per
// device (a process may drive several GPUs)
void set_p1_smem() {
    static std::mutex mu;
    static uint64_t done_mask[4] = {0, 0, 0, 0};  // devices 0..255
    int dev = 0;
    cudaGetDevice(&dev);
    dev = std::max(0, std::min(dev, 255));
    std::lock_guard<std::mutex> g(mu);
    if (done_mask[dev >> 6] & (1ull << (dev & 63))) return;
    cudaFuncSetAttribute(k_pass2_gr<G2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, P2R_SMEM);
    cudaFuncSetAttribute(k_pass2_gr<G2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, P2R_SMEM);
    cudaFuncSetAttribute(k_pass1_gauss<false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, P1_SMEM_OCC2);
    cudaFuncSetAttribute(k_pass1_gauss<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, P1_SMEM_OCC2);
    cudaFuncSetAttribute(k_pass1_gauss<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, P1_SMEM_OCC2);
    cudaFuncSetAttribute(k_pass1_gauss<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, P1_SMEM_OCC2);
    cudaFuncSetAttribute(k_pass1_gauss<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, P1_SMEM_OCC2);
    cudaFuncSetAttribute(k_pass1_gauss<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, P1_SMEM_OCC2);
    cudaFuncSetAttribute(k_pass1_gauss<false, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, P1_SMEM_OCC2);
    cudaFuncSetAttribute(k_pass1_gauss<true, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, P1_SMEM_OCC2);
    cudaFuncSetAttribute(k_pass1_box<G1, R_ANCHOR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         P1_SMEM);
    done_mask[dev >> 6] |= 1ull << (dev & 63);
}


// Pass-2 x-chunking of one batch's launch: equal chunks when rows x groups
// cannot fill the GPU (fitted heuristic), or for the device entry's
// single-batch runs of a few waves the planned unequal split (p2_plan_split,
// at most 3 chunks, costliest first).  `ngroups` thread groups of G2 terms,
// `npart` k_pass2_gr group blocks.
struct P2Plan {
    int nchunk, tiles_per_chunk, warm_tiles;
    int xlpt, xb1, xb2, xord;
};
P2Plan p2_chunk_plan(const Layout& L, const tbf_spatial* sp, int ngroups, int npart,
                     bool hpipe, int nrb_run = -1) {
    const bool box = sp->kind == TBF_SPATIAL_BOX;
    // 128-row blocks in flight: the whole image, or the host entry's output
    // bands (nrb_run)
    const int B = L.B, nrb = nrb_run > 0 ? nrb_run : (L.H + P2_THREADS - 1) / P2_THREADS;
    P2Plan pp{};
    int nchunk = 1;
    pp.warm_tiles = (std::max(sp->ext_x, 1) + TILE - 1) / TILE;
    if (box) {
        const long long threads = (long long)nrb * P2_THREADS * ngroups * B;
        const long long target = 148LL * 12 * 32 * 3 / 2;
        const int win = 2 * sp->radius + 1;
        while (threads * nchunk < target && nchunk < 64) {
            const int cols = (L.ntx + 2 * nchunk - 1) / (2 * nchunk) * TILE;
            if (cols < 4 * win) break;  // window init <= 25% of a chunk
            nchunk *= 2;
        }
    } else if (g_p2_chunks > 0) {
        nchunk = std::min(g_p2_chunks, L.ntx);
    } else {
        const long long threads = (long long)nrb * P2_THREADS * ngroups * B;
        const long long target = 148LL * 12 * 32 * 3 / 2;  // ~1.5 waves of 12 warps/SM
        const long long wave = 148LL * 12 * 32;
        // measured: G=4 prefers fewer, longer rows unless the GPU is far from full
        const int max_chunks = 64;
        while (threads * nchunk < target && nchunk < max_chunks) {
            const int tpc = (L.ntx + 2 * nchunk - 1) / (2 * nchunk);
            // warm-up <= 25% of a chunk; below one wave (latency-bound small
            // images) accept warm-up up to the chunk length
            const bool ok = tpc >= 4 * pp.warm_tiles || (threads * nchunk < wave && tpc >= pp.warm_tiles);
            if (!ok) break;
            nchunk *= 2;
        }
        // launches of several waves of k_pass2_gr blocks: the last wave runs
        // partly empty, so a chunk count whose block count fills the waves
        // better can pay for its warm-up tiles.  Cost = waves rounded up x
        // tiles a block walks (its chunk plus the warm-up); a count wins by
        // >= 3%.  Config 5 (1536 blocks, 3.46 waves): 2 chunks, pass 2 -5%
        // measured (profiles/sweep_p2_chunks_r02.log)
        if (npart > 0 && nchunk == 1 && threads >= wave) {
            const long long blocks1 = (long long)nrb * (P2_THREADS / 32) * npart * B;
            const long long slots = 148LL * TBF_P2_MINB;
            auto cost = [&](int n) {
                const int tpc = (L.ntx + n - 1) / n;
                const long long waves = (blocks1 * n + slots - 1) / slots;
                return (double)waves * (tpc + (n > 1 ? pp.warm_tiles : 0));
            };
            const double c1 = cost(1);
            double best = c1;
            for (int n = 2; n <= 4; ++n) {
                if ((L.ntx + n - 1) / n < 4 * pp.warm_tiles) break;
                const double c = cost(n);
                if (c < best && c < 0.97 * c1) {
                    best = c;
                    nchunk = n;
                }
            }
        }
    }
    pp.tiles_per_chunk = (L.ntx + nchunk - 1) / nchunk;
    nchunk = (L.ntx + pp.tiles_per_chunk - 1) / pp.tiles_per_chunk;
    pp.nchunk = nchunk;
    if (box || L.nb != 1) return pp;
    // unequal x-chunks (at most 3), costliest first: the development override
    // TBF_P2_XSPLIT (widths in tiles, left to right), else the planner for
    // launches of a few waves (device entry only: the host entry's band
    // launches want short blocks, measured +14%)
    std::vector<int> b;
    const char* ev = getenv("TBF_P2_XSPLIT");
    if (ev && *ev) {
        b.push_back(0);
        for (const char* q = ev; *q && b.size() < 4 && b.back() < L.ntx;) {
            int v = std::max(1, (int)strtol(q, (char**)&q, 10));
            if (*q == ',') ++q;
            b.push_back((!*q || b.size() == 3) ? L.ntx : std::min(L.ntx, b.back() + v));
        }
        if (b.back() < L.ntx) b.back() = L.ntx;
    } else if (g_p2_chunks <= 0 && (g_lpt_split & 2) && (!hpipe || (g_lpt_split & 8))) {
        const int slots = 148 * 3;  // k_pass2_gr blocks resident per SM
        const long long per_chunk = (long long)nrb * (P2_THREADS / 32) * npart * B;
        if (per_chunk < 6LL * slots && 2 * per_chunk >= slots && L.ntx >= 8) {
            b = p2_plan_split(L.ntx, pp.warm_tiles, nchunk, per_chunk, slots);
            bool equal = (int)b.size() - 1 == nchunk;  // the planner kept the equal split
            for (int c = 0; equal && c <= nchunk; ++c) equal = b[c] == std::min(L.ntx, c * pp.tiles_per_chunk);
            if (equal || b.size() > 4) b.clear();
        }
    }
    if (b.size() >= 3) {
        pp.nchunk = (int)b.size() - 1;
        pp.xlpt = 1;
        pp.xb1 = b[1];
        pp.xb2 = pp.nchunk > 2 ? b[2] : L.ntx;
        std::vector<std::pair<double, int>> cs;
        for (int c = 0; c < pp.nchunk; ++c) cs.push_back({-p2_chunk_cost(b[c], b[c + 1], L.ntx, pp.warm_tiles), c});
        std::stable_sort(cs.begin(), cs.end());
        for (int r = 0; r < pp.nchunk; ++r) pp.xord |= cs[r].second << (2 * r);
    }
    return pp;
}

// Pass-1 instantiation for a layout: 2 planned chunks; 1 equal chunks whose
// interior warm-up rows are at least a tenth of the column (config 1: 62%,
// 2.8% faster); else 0, the original code (config 5's batches, 2 chunks of
// 8192 rows with 2% warm-up rows, lost 7% in mode 1 to its spills)
int p1_mode(const Layout& L, const Pass1Args& p1) {
    if (p1.ylpt) return 2;
    return (L.nyc > 1 && 10LL * L.ywarm * (L.nyc - 1) >= L.H) ? 1 : 0;
}

// pdl: programmatic dependent launch on the previous pass-1 launch of the
// stream (the host entry's column strips): this launch's blocks may start
// once every block of the previous one is running (each signals at its
// start), so strip s+1 fills the slots strip s frees instead of waiting for
// its tail.  Safe with the x chain: strip s+1's blocks wait only for strip
// s's, which are all resident by then.
void launch_pass1(bool fold, int mode, dim3 grid, int smem, cudaStream_t st, const Pass1Args& p1,
                  bool pdl = false) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(P1_WARPS * 32);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (p1.cs > 1) {  // clusters of p1.cs consecutive stripes (grid.x is a multiple)
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = (unsigned)p1.cs;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    switch (mode * 2 + (fold ? 1 : 0)) {
        case 0: cudaLaunchKernelEx(&cfg, k_pass1_gauss<false, 0>, p1); break;
        case 1: cudaLaunchKernelEx(&cfg, k_pass1_gauss<true, 0>, p1); break;
        case 2: cudaLaunchKernelEx(&cfg, k_pass1_gauss<false, 1>, p1); break;
        case 3: cudaLaunchKernelEx(&cfg, k_pass1_gauss<true, 1>, p1); break;
        case 4: cudaLaunchKernelEx(&cfg, k_pass1_gauss<false, 2>, p1); break;
        default: cudaLaunchKernelEx(&cfg, k_pass1_gauss<true, 2>, p1); break;
    }
}

void launch_pass1_zero(bool fold, dim3 grid, int smem, cudaStream_t st, const Pass1Args& p1) {
    if (fold)
        k_pass1_gauss<true, 0, true><<<grid, P1_WARPS * 32, smem, st>>>(p1);
    else
        k_pass1_gauss<false, 0, true><<<grid, P1_WARPS * 32, smem, st>>>(p1);
}

// Core driver: pairs [tbeg, tend) in batches of L.tb terms.  Either
// accumulates into caller num/den (row-major), or (out != null) writes the
// guarded ratio.
// Split [0, n) into k parts with quadratically growing (grow = true) or
// shrinking sizes: the first input strip / last output band are small, so
// the copies left exposed at the two ends of the host pipeline are short.
std::vector<int> quad_split(int n, int k, bool grow) {
    std::vector<int> b{0};
    k = std::max(1, std::min(k, n));
    for (int i = 1; i < k; ++i) {
        const double u = (double)i / k;
        const double frac = grow ? u * u : 1.0 - (1.0 - u) * (1.0 - u);
        const int v = std::max(b.back() + 1, std::min(n - (k - i), (int)std::lround(frac * n)));
        b.push_back(v);
    }
    b.push_back(n);
    return b;
}

// Host-buffer I/O of tbf_bilateral_trig_host: f and out are device buffers,
// h_f / h_out the caller's host arrays.
struct HostIO {
    const float* h_f;
    float* h_out;
    int strips;  // column strips: H2D of strip s+1 overlaps pass 1 of strip s
    int bands;   // row bands: D2H of band b overlaps pass 2 of band b+1
};

// Pinned staging of the per-call term table (see run_terms).
constexpr size_t TAB_CACHE = 64;
struct TabEntry {
    uint64_t hash;
    std::vector<float> content;
    float* pinned;
    cudaEvent_t last_use;
    uint64_t tick;
};

uint64_t fnv1a(const std::vector<float>& v) {
    uint64_t h = 1469598103934665603ull;
    const unsigned char* p = reinterpret_cast<const unsigned char*>(v.data());
    for (size_t i = 0; i < v.size() * sizeof(float); ++i) h = (h ^ p[i]) * 1099511628211ull;
    return h;
}

int stage_term_table(const std::vector<float>& h_tab, float* d_tab, cudaStream_t st) {
    static std::mutex mu;
    static std::vector<TabEntry> cache;
    static uint64_t clock = 0;
    std::lock_guard<std::mutex> g(mu);
    const uint64_t h = fnv1a(h_tab);
    TabEntry* e = nullptr;
    for (auto& c : cache)
        if (c.hash == h && c.content == h_tab) e = &c;
    if (!e) {
        if (cache.size() >= TAB_CACHE) {  // evict the least recently used entry
            auto lru = std::min_element(cache.begin(), cache.end(),
                                        [](const TabEntry& a, const TabEntry& b) { return a.tick < b.tick; });
            cudaEventSynchronize(lru->last_use);  // its last copy has read the buffer
            cudaEventDestroy(lru->last_use);
            cudaFreeHost(lru->pinned);
            cache.erase(lru);
        }
        float* p = nullptr;
        if (cudaHostAlloc(&p, h_tab.size() * 4, cudaHostAllocDefault) != cudaSuccess)
            return fail(TBF_ERR_CUDA, "pinned term table: %s", cudaGetErrorString(cudaGetLastError()));
        std::copy(h_tab.begin(), h_tab.end(), p);
        cudaEvent_t ev;
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        cache.push_back(TabEntry{h, h_tab, p, ev, 0});
        e = &cache.back();
    }
    e->tick = ++clock;
    cudaMemcpyAsync(d_tab, e->pinned, h_tab.size() * 4, cudaMemcpyHostToDevice, st);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusNone) cudaEventRecord(e->last_use, st);
    return check_cuda("term table copy");
}

int run_terms(const float* f, float* num, float* den, float* out, int B, int H, int W,
              const tbf_spatial* sp, const tbf_terms* terms, int tbeg, int tend, int batch_terms,
              int accumulate, void* ws, size_t ws_bytes, unsigned long long* counters,
              cudaStream_t st, const HostIO* hio = nullptr, int row0 = 0, int row1 = -1) {
    int rc = validate(sp, terms, tbeg, tend);
    if (rc) return rc;
    const int nrange = tend - tbeg;
    Layout L;
    rc = make_layout(B, H, W, sp, nrange, batch_terms, &L, (hio == nullptr || (g_lpt_split & 4)) ? 1 : 0,
                     row0, row1);
    if (rc) return rc;
    const bool band = L.row0 > 0 || L.row1 < H;
    if (band && (out || hio || sp->kind == TBF_SPATIAL_BOX))
        return fail(TBF_ERR_PARAM, "row bands are for the recursive partial (num/den) path only");
    if (!ws || ws_bytes < L.total)
        return fail(TBF_ERR_WORKSPACE, "workspace too small: need %zu have %zu", L.total, ws_bytes);
    char* w8 = (char*)ws;
    float* fT = (float*)(w8 + L.off_fT);
    float* fY = (float*)(w8 + L.off_fY);
    float* tab = (float*)(w8 + L.off_tab);
    auto slot = [&](int k, size_t off) { return (float*)(w8 + L.off_slot + (size_t)(k % L.nslot) * L.slot_bytes + off); };
    const bool box = sp->kind == TBF_SPATIAL_BOX;
    const int nb = L.nb;
    if (out && nb > 1) {  // accumulate batches in workspace num/den, ratio at the end
        num = (float*)(w8 + L.off_num);
        den = (float*)(w8 + L.off_den);
        accumulate = 0;
    }
    // streams: pass 1 on the caller's stream, the rest of each batch on an
    // internal stream when pipelining (joined back before returning)
    cudaStream_t s2 = (L.nslot > 1) ? aux_stream() : st;
    if (!s2) s2 = st;
    std::vector<cudaEvent_t> ev_done(nb, nullptr);

    // term tables: nu split hi/lo, float weights; zero padded past the end
    const int ld = nrange + TAB_PAD;
    double Rx[16] = {0}, MW[16] = {0};
    std::vector<float> bx, hx;
    int nHx = 0;
    if (!box) {
        right_ext_coeffs(sp, L.Ex, Rx, bx);
        left_response(sp, W, hx, nHx, MW);
    }
    std::vector<float> h_tab(tab_bx_offset(nrange) + bx.size() + hx.size(), 0.f);
    std::copy(bx.begin(), bx.end(), h_tab.begin() + tab_bx_offset(nrange));
    std::copy(hx.begin(), hx.end(), h_tab.begin() + tab_bx_offset(nrange) + bx.size());
    for (int j = 0; j < nrange; ++j) {
        double nu = terms->nu[tbeg + j];
        float hi = (float)nu;
        h_tab[j] = hi;
        h_tab[ld + j] = (float)(nu - (double)hi);
        h_tab[2 * ld + j] = (float)terms->weight[tbeg + j];
    }
    // the table is copied from a pinned buffer per distinct table content, so
    // a call captured in a CUDA graph replays the copy of exactly the table it
    // was captured with.  The cache is bounded (LRU, TAB_CACHE entries): an
    // evicted buffer is freed only after the event recorded behind its last
    // copy has completed (a graph capture is the caller's to keep within the
    // bound: more distinct live tables than TAB_CACHE would recycle buffers)
    {
        if ((rc = stage_term_table(h_tab, tab, st))) return rc;
    }

    // host input: column strips copied on an internal stream; pass 1 of the
    // first batch runs strip by strip as they land (columns are independent
    // in pass 1), the range check and transpose once the whole input is in
    const bool hpipe = hio && !box && L.nslot == 1 && out;
    // pass-1 thread-block clusters: the largest of TBF_OPT_P1_CLUSTER, 2, 1
    // stripes that divides the stripe count (cluster hand-offs go through
    // DSMEM, only the hand-offs between clusters through L2)
    int p1cs = 1;
    if (!box)
        for (int c = std::min(std::max(g_p1_cluster, 1), 8); c > 1; c /= 2)
            if (L.nst % c == 0) {
                p1cs = c;
                break;
            }
    std::vector<cudaEvent_t> ev_strip;
    std::vector<int> sb{0, L.nst};  // strip boundaries in stripes (P1_WARPS column tiles)
    cudaEvent_t e_ready = nullptr;
    if (hio) {
        cudaStream_t sh = aux_stream(1);
        if (!sh) return fail(TBF_ERR_CUDA, "no copy stream");
        e_ready = event_get();
        cudaEventRecord(e_ready, st);  // term table queued, earlier users of f done
        cudaStreamWaitEvent(sh, e_ready, 0);
        if (hpipe) {  // in whole clusters of stripes
            sb = quad_split(L.nst / p1cs, hio->strips, true);
            for (int& v : sb) v *= p1cs;
        }
        float* df = const_cast<float*>(f);
        for (size_t s = 0; s + 1 < sb.size(); ++s) {
            const int x0 = sb[s] * STRIPE;
            const int cols = std::min(W, sb[s + 1] * STRIPE) - x0;
            {
                Prof pr(KK_H2D, sh);
                cudaMemcpy2DAsync(df + x0, (size_t)W * 4, hio->h_f + x0, (size_t)W * 4, (size_t)cols * 4,
                                  (size_t)B * H, cudaMemcpyHostToDevice, sh);
            }
            ev_strip.push_back(event_get());
            cudaEventRecord(ev_strip.back(), sh);
        }
        // with strip-wise pass 1 the caller's stream waits for each strip's
        // transpose instead (below), so pass 1 starts on the first strip
        if (!(hpipe && ev_strip.size() > 1)) cudaStreamWaitEvent(st, ev_strip.back(), 0);
        if ((rc = check_cuda("host to device"))) return rc;
    }

    // transpose, fused with the input range check in the full filter
    // (tbf_bilateral_trig / _host); the sharded path checks separately.  With
    // host strips, each strip is transposed on its own stream before its pass 1.
    const bool strip_p1 = hpipe && ev_strip.size() > 1;
    unsigned long long* const rc_counters = out ? counters : nullptr;
    if (!strip_p1) {
        dim3 tgrid((W + TILE - 1) / TILE, (H + TILE - 1) / TILE, B);
        Prof pr(KK_TRANSPOSE, st);
        k_transpose<<<tgrid, 256, 0, st>>>(f, fT, fY, H, W, -1e-9, terms->T + 1e-9, rc_counters, 0);
    }
    if ((rc = check_cuda("transpose"))) return rc;

    set_p1_smem();
    const Casc kc = to_casc(sp);
    // fold the y-sweep scale into the weights when the unscaled intermediates
    // (up to ~T / g^4) stay far below FLT_MAX
    // (measured: ~1% faster on configs 2-4 now that it no longer spills)
    const bool fold = g_pass1_fold && !box &&
                      std::log10(std::max(terms->T, 1.0)) - 4.0 * std::log10(sp->g1 * sp->g2) < 34.0;
    if (s2 != st) {
        cudaEvent_t e0 = event_get();
        cudaEventRecord(e0, st);  // f, fT and the term table are ready
        cudaStreamWaitEvent(s2, e0, 0);
    }
    for (int bi = 0; bi < nb; ++bi) {
        const int jb = bi * L.tb;
        const int n = std::min(L.tb, nrange - jb);
        float* ckpt = slot(bi, L.s_ckpt);
        float* floc = slot(bi, L.s_floc);
        float* mail = slot(bi, L.s_mail);
        int* flags = reinterpret_cast<int*>(slot(bi, L.s_flags));
        const size_t nflags = (size_t)L.tb * B * L.nst * ((H + TILE - 1) / TILE);
        unsigned int* tickets = reinterpret_cast<unsigned int*>(flags + nflags);
        float* edge = slot(bi, L.s_edge);
        float* s0 = slot(bi, L.s_s0);
        float* bst = slot(bi, L.s_bst);
        float* part = slot(bi, L.s_part);
        // the slot is free once batch bi - nslot has finished on s2
        if (s2 != st && bi >= L.nslot) cudaStreamWaitEvent(st, ev_done[bi - L.nslot], 0);
        TermDev td;
        td.nu_hi = tab + jb;
        td.nu_lo = tab + ld + jb;
        td.w = tab + 2 * ld + jb;
        td.dnu = (float)terms->dnu;
        td.n = n;
        td.anchor = R_ANCHOR;
        // the zero frequency (first pair of an even N) as the packed 1-plane
        // unit: its own pass 1 (k_pass1_gauss<.., ZU>) and pass 2
        // (k_pass2_zero) on a side stream; the main launches take the rest.
        // Needs every row quarter's warm-up inside the image (Ey = K <= hq)
        const bool zu = !box && !band && g_zero_unit && jb == 0 && terms->nu[tbeg] == 0.0 && H >= 4 * TILE &&
                        L.Ey == sp->ext_y && L.Ey <= L.zhq && H >= L.Ey + 4 * TILE;
        const int term0 = zu ? 1 : 0;
        const int nmain = n - term0;
        cudaStream_t zs = zu ? aux_stream(5) : nullptr;

        Pass1Args p1;
        p1.f = f;
        p1.fY = fY;
        p1.B = B;
        p1.H = H;
        p1.W = W;
        p1.Ey = L.Ey;
        p1.nseg = L.nseg;
        p1.nyc = L.nyc;
        p1.ych_rows = L.ych_rows;
        p1.ylpt = L.ych_lpt;
        p1.yb1 = L.nyc > 1 ? L.ychb[1] : H;
        p1.yb2 = L.nyc > 2 ? L.ychb[2] : H;
        p1.ywarm = L.ywarm;
        p1.row0 = L.row0;
        p1.row1 = L.row1;
        p1.Ex = L.Ex;
        p1.ne = L.ne;
        p1.edge_all = L.edge_all;
        p1.ntx = L.ntx;
        p1.nst = L.nst;
        p1.st0 = 0;
        p1.nst_run = L.nst;
        p1.term0 = term0;
        p1.nterm = nmain;
        p1.cs = p1cs;
        p1.hq = L.zhq;
        // the zero unit's virtual rows in chunks about as long as the main
        // ones (its blocks then run beside the main pass 1), at most nyc
        // (checkpoint slots)
        p1.zyc = std::max(1, std::min(L.nyc, (L.zhq + std::max(L.ych_rows, L.ywarm) - 1) / std::max(L.ych_rows, L.ywarm)));
        p1.zrows = ((L.zhq + p1.zyc - 1) / p1.zyc + TILE - 1) / TILE * TILE;
        p1.zyc = (L.zhq + p1.zrows - 1) / p1.zrows;
        p1.k = kc;
        p1.t = td;
        p1.ckpt = ckpt;
        p1.floc = floc;
        p1.mail = mail;
        p1.flags = flags;
        p1.nsegH = (H + TILE - 1) / TILE;
        p1.edge = edge;
        // box: blocks of P1_WARPS terms x one column tile; Gaussian: blocks
        // of one term x one stripe (term fastest, then stripe, y-chunk)
        const dim3 gbox(L.ntx, (n + P1_WARPS - 1) / P1_WARPS, B);
        // Gaussian: 1-D grid, blocks map to (stripe, frame, y-chunk, term) by a
        // dispatch ticket; one counter per launch after the flags
        auto p1grid = [&](int nst_run) { return dim3(nst_run * B * L.nyc * nmain, 1, 1); };
        const int p1smem = g_p1_occ == 2 ? P1_SMEM_OCC2 : P1_SMEM_GAUSS;
        if (!box) cudaMemsetAsync(flags, 0, (nflags + P1_MAX_LAUNCHES) * sizeof(int), st);
        cudaEvent_t e_zu_ready = nullptr;
        if (zu) {  // flags cleared (and, without host strips, f transposed)
            e_zu_ready = event_get();
            cudaEventRecord(e_zu_ready, st);
        }
        if (strip_p1 && bi == 0 && nmain == 0) {
            // only the zero unit: the whole input must be in before it starts
            for (size_t s = 0; s < ev_strip.size(); ++s) {
                const int t0 = sb[s] * P1_WARPS, t1 = std::min(L.ntx, sb[s + 1] * P1_WARPS);
                dim3 tg(t1 - t0, (H + TILE - 1) / TILE, B);
                cudaStreamWaitEvent(st, ev_strip[s], 0);
                Prof pr(KK_TRANSPOSE, st);
                k_transpose<<<tg, 256, 0, st>>>(f, fT, fY, H, W, -1e-9, terms->T + 1e-9, rc_counters, t0);
            }
            e_zu_ready = event_get();
            cudaEventRecord(e_zu_ready, st);
        } else if (strip_p1 && bi == 0) {
            // strip s: transpose (+ range check) on a side stream as soon as
            // its copy lands, pass 1 in strip order on the caller's stream
            // (stripe s waits for stripe s-1: a strip's blocks only wait for
            // strips launched before it on the same stream)
            cudaStream_t ts = aux_stream(2);
            cudaStreamWaitEvent(ts, e_ready, 0);
            for (size_t s = 0; s < ev_strip.size(); ++s) {
                cudaStreamWaitEvent(ts, ev_strip[s], 0);
                p1.st0 = sb[s];
                p1.nst_run = sb[s + 1] - sb[s];
                {
                    const int t0 = sb[s] * P1_WARPS, t1 = std::min(L.ntx, sb[s + 1] * P1_WARPS);
                    dim3 tg(t1 - t0, (H + TILE - 1) / TILE, B);
                    Prof pr(KK_TRANSPOSE, ts);
                    k_transpose<<<tg, 256, 0, ts>>>(f, fT, fY, H, W, -1e-9, terms->T + 1e-9, rc_counters, t0);
                }
                cudaEvent_t e = event_get();
                cudaEventRecord(e, ts);
                cudaStreamWaitEvent(st, e, 0);
                p1.ticket = tickets + std::min<size_t>(s, P1_MAX_LAUNCHES - 2);  // (the last is the zero unit's)
                {
                    Prof pr(KK_PASS1, st);
                    launch_pass1(fold, p1_mode(L, p1), p1grid(p1.nst_run), p1smem, st, p1, s > 0);
                }
            }
            p1.st0 = 0;
            p1.nst_run = L.nst;
            if (zu) {  // the zero unit reads every strip: after the last transpose
                cudaEvent_t e_t = event_get();
                cudaEventRecord(e_t, ts);
                cudaStreamWaitEvent(zs, e_t, 0);
            }
        } else if (nmain > 0) {
            p1.ticket = tickets;
            Prof pr(KK_PASS1, st);
            if (box)
                k_pass1_box<G1, R_ANCHOR><<<gbox, P1_WARPS * 32, P1_SMEM, st>>>(p1, sp->radius);
            else
                launch_pass1(fold, p1_mode(L, p1), p1grid(L.nst), p1smem, st, p1);
        }
        if (zu) {
            cudaStreamWaitEvent(zs, e_zu_ready, 0);
            Pass1Args pz = p1;
            pz.term0 = 0;
            pz.nterm = 1;
            pz.st0 = 0;
            pz.nst_run = L.nst;
            pz.ticket = tickets + (P1_MAX_LAUNCHES - 1);
            pz.cs = 1;
            {
                Prof pr(KK_PASS1, zs);
                launch_pass1_zero(fold, dim3(L.nst * B * pz.zyc), p1smem, zs, pz);
            }
            cudaEvent_t e_z1 = event_get();
            cudaEventRecord(e_z1, zs);
            cudaStreamWaitEvent(st, e_z1, 0);  // joined before the edge kernel
        }
        if ((rc = check_cuda("pass1"))) return rc;
        if (s2 != st) {  // hand the batch to the second stream
            cudaEvent_t e1 = event_get();
            cudaEventRecord(e1, st);
            cudaStreamWaitEvent(s2, e1, 0);
        }

        if (!box) {
            EdgeArgs ea;
            ea.B = B;
            ea.H = H;
            ea.W = W;
            ea.row0 = L.row0;
            ea.row1 = L.row1;
            ea.Ex = L.Ex;
            ea.ne = L.ne;
            ea.edge_all = L.edge_all;
            ea.nst = L.nst;
            ea.k = kc;
            ea.n = n;
            ea.edge = edge;
            ea.mail = mail;
            for (int q = 0; q < 16; ++q) {
                ea.MW[q] = (float)MW[q];
                ea.Rx[q] = (float)Rx[q];
            }
            ea.bx = reinterpret_cast<const float4*>(tab + tab_bx_offset(nrange));
            ea.s0 = s0;
            ea.bstate = bst;
            dim3 gc((L.row1 - L.row0 + 127) / 128, n * B);
            { Prof pr(KK_CHAIN, s2); k_edge<<<gc, 128, 0, s2>>>(ea); }
            if ((rc = check_cuda("edge"))) return rc;
        }

        Pass2Args p2;
        p2.fT = fT;
        p2.B = B;
        p2.H = H;
        p2.W = W;
        p2.ntx = L.ntx;
        p2.k = kc;
        p2.t = td;
        // pass 2: the block-summed variant (k_pass2_gr) for the Gaussian, over
        // the terms after the zero unit when it has its own pass 2
        p2.term0 = term0;
        const int npart = box ? -1 : (((nmain + G2 - 1) / G2 + P2R_GR - 1) / P2R_GR);
        p2.ngroups = (nmain + G2 - 1) / G2;
        {
            const double g = sp->g1 * sp->g2;
            p2.wscale = box ? 1.f : (float)(fold ? g * g * g * g : g * g);
        }
        p2.floc = floc;
        p2.nHx = nHx;
        p2.Hx = reinterpret_cast<const float4*>(tab + tab_bx_offset(nrange) + bx.size());
        p2.s0 = s0;
        p2.bstate = bst;
        p2.part = part;
        p2.order = g_p2_order;
        // x-chunking of pass-2 rows (p2_chunk_plan)
        const int nrb = (H + P2_THREADS - 1) / P2_THREADS;
        const P2Plan pp = p2_chunk_plan(L, sp, p2.ngroups, npart, hpipe);
        int nchunk = pp.nchunk;
        p2.warm_tiles = pp.warm_tiles;
        p2.tiles_per_chunk = pp.tiles_per_chunk;
        p2.xlpt = pp.xlpt;
        p2.xb1 = pp.xb1;
        p2.xb2 = pp.xb2;
        p2.xord = pp.xord;
        if (pp.xlpt) p2.order = 4;
        // the zero unit's pass 2 on its side stream, after the edge kernel;
        // every reduce below waits for it
        const size_t xpl = xm_plane(B, W, H);
        cudaEvent_t e_z2 = nullptr;
        if (zu) {
            cudaEvent_t e_e = event_get();
            cudaEventRecord(e_e, s2);
            cudaStreamWaitEvent(zs, e_e, 0);
            ZeroArgs za;
            za.B = B;
            za.H = H;
            za.W = W;
            za.ntx = L.ntx;
            za.hq = L.zhq;
            za.term = 0;
            za.k = kc;
            za.warm_tiles = pp.warm_tiles;
            // x-chunks until ~2 waves of threads (warm-ups of >= K per chunk)
            int zch = 1;
            while ((long long)L.zhq * B * zch < 148LL * 12 * 32 * 2 && zch * 2 <= std::max(1, L.ntx / std::max(1, 2 * pp.warm_tiles)))
                zch *= 2;
            za.tiles_per_chunk = (L.ntx + zch - 1) / zch;
            zch = (L.ntx + za.tiles_per_chunk - 1) / za.tiles_per_chunk;
            za.wt = (float)terms->weight[tbeg] * p2.wscale;
            za.floc = floc;
            za.nHx = nHx;
            za.Hx = p2.Hx;
            za.s0 = s0;
            za.bstate = bst;
            za.num = part + (size_t)npart * 2 * xpl;
            {
                Prof pr(KK_PASS2, zs);
                k_pass2_zero<<<dim3((L.zhq + 127) / 128, zch, B), 128, 0, zs>>>(za);
            }
            if ((rc = check_cuda("pass2 zero unit"))) return rc;
            e_z2 = event_get();
            cudaEventRecord(e_z2, zs);
        }
        ReduceArgs ra;
        ra.part = part;
        ra.ngroups = box ? p2.ngroups : npart;
        ra.zpart = zu ? part + (size_t)npart * 2 * xpl : nullptr;
        ra.den_add = zu ? (float)terms->weight[tbeg] : 0.f;
        ra.B = B;
        ra.H = H;
        ra.W = W;
        ra.f = f;
        ra.counters = counters;
        ra.i_base = 0;
        const bool add = bi > 0 || (accumulate && !out);
        ra.in_num = add ? num : nullptr;
        ra.in_den = add ? den : nullptr;
        const bool last = bi == nb - 1;
        if (out && last) {
            ra.num = nullptr;
            ra.den = nullptr;
            ra.out = out;
        } else {
            ra.num = num;
            ra.den = den;
            ra.out = nullptr;
        }
        // pass 2 + reduce over 128-row blocks [rb0, rb0 + nrb_run) on stream q
        auto pass2_reduce = [&](int rb0, int nrun, cudaStream_t q) -> int {
            p2.rb0 = rb0;
            p2.nrb_run = nrun;
            dim3 g2(nrun * nchunk, p2.ngroups, B);
            if (nmain > 0) {
                Prof pr(KK_PASS2, q);
                if (box)
                    k_pass2_box<G2, R_ANCHOR><<<g2, P2_THREADS, 0, q>>>(p2, sp->radius);
                else if (p2.xlpt)
                    k_pass2_gr<G2, true><<<dim3(nrun * (P2_THREADS / 32) * nchunk * npart, 1, B), 32 * P2R_GR,
                                           P2R_SMEM, q>>>(p2);
                else
                    k_pass2_gr<G2, false><<<dim3(nrun * (P2_THREADS / 32) * nchunk, npart, B), 32 * P2R_GR,
                                            P2R_SMEM, q>>>(p2);
            }
            int e;
            if ((e = check_cuda("pass2"))) return e;
            ra.i_base = rb0 * P2_THREADS;  // RED_I == P2_THREADS
            if (e_z2) cudaStreamWaitEvent(q, e_z2, 0);
            {
                const int rows = std::min(H - ra.i_base, nrun * P2_THREADS);
                dim3 rgrid((W + TILE - 1) / TILE, (rows + RED_I - 1) / RED_I, B);
                Prof pr(KK_REDUCE, q);
                k_reduce<<<rgrid, 256, 0, q>>>(ra);
            }
            return check_cuda("reduce");
        };
        if (hpipe && last && hio->bands > 1 && nrb > 1) {
            // row bands on alternating streams; each band's rows go back to the
            // host while the next band filters
            // equal bands (in 128-row blocks): the copy-back is about as long
            // as the last pass 2, so it must start early and keep pace; each
            // band's pass 2 gets x-chunks for its own (two bands') rows
            std::vector<int> bb{0};
            const int nbands = std::max(1, std::min(hio->bands, nrb));
            for (int k = 1; k <= nbands; ++k) bb.push_back((int)((long long)nrb * k / nbands));
            cudaStream_t sd = aux_stream(4);
            cudaEvent_t e_c = event_get();
            cudaEventRecord(e_c, s2);  // edge kernel and everything before it
            for (size_t k = 0; k + 1 < bb.size(); ++k) {
                const int rb0 = bb[k], nrun = bb[k + 1] - bb[k];
                cudaStream_t q = aux_stream(2 + (int)(k & 1));
                cudaStreamWaitEvent(q, e_c, 0);
                if (!box) {
                    const P2Plan bp = p2_chunk_plan(L, sp, p2.ngroups, npart, true, 2 * nrun);
                    nchunk = bp.nchunk;
                    p2.tiles_per_chunk = bp.tiles_per_chunk;
                    p2.warm_tiles = bp.warm_tiles;
                    p2.xlpt = 0;
                    p2.order = g_p2_order;
                }
                if ((rc = pass2_reduce(rb0, nrun, q))) return rc;
                cudaEvent_t e_r = event_get();
                cudaEventRecord(e_r, q);
                cudaStreamWaitEvent(sd, e_r, 0);
                const int r0 = rb0 * P2_THREADS;
                const int r1 = std::min(H, (rb0 + nrun) * P2_THREADS);
                Prof pr(KK_D2H, sd);
                cudaMemcpy2DAsync(hio->h_out + (size_t)r0 * W, (size_t)H * W * 4, out + (size_t)r0 * W,
                                  (size_t)H * W * 4, (size_t)(r1 - r0) * W * 4, B, cudaMemcpyDeviceToHost, sd);
            }
            cudaEvent_t e_d = event_get();
            cudaEventRecord(e_d, sd);
            cudaStreamWaitEvent(st, e_d, 0);  // join (sd waited on every band)
            if ((rc = check_cuda("device to host"))) return rc;
            hio = nullptr;  // output delivered
        } else {
            const int rb0 = L.row0 / P2_THREADS, rb1 = (L.row1 + P2_THREADS - 1) / P2_THREADS;
            if ((rc = pass2_reduce(rb0, rb1 - rb0, s2))) return rc;
        }
        if (s2 != st) {
            ev_done[bi] = event_get();
            cudaEventRecord(ev_done[bi], s2);
        }
    }
    if (s2 != st) cudaStreamWaitEvent(st, ev_done[nb - 1], 0);  // join
    if (hio && out) {  // host output not yet delivered (no banding)
        cudaMemcpyAsync(hio->h_out, out, (size_t)B * H * W * 4, cudaMemcpyDeviceToHost, st);
        if ((rc = check_cuda("device to host"))) return rc;
    }
    return TBF_OK;
}

template <typename T>
int bilateral_direct_impl(const T* f, int32_t B, int32_t H, int32_t W, const int32_t* samples, int64_t n,
                          const double* taps, int32_t radius, int32_t range_kind, double range_param,
                          int32_t degree, double* out, unsigned long long* d_counters, void* stream) {
    if (B < 1 || H < 1 || W < 1) return fail(TBF_ERR_DIM, "bad shape B=%d H=%d W=%d", B, H, W);
    if (radius < 0 || !taps) return fail(TBF_ERR_PARAM, "bad window (radius %d)", radius);
    if (range_kind != 0 && range_kind != 1) return fail(TBF_ERR_PARAM, "unknown range kind %d", range_kind);
    if (range_kind == 0 && !(range_param > 0.0)) return fail(TBF_ERR_PARAM, "sigma_r must be positive");
    if (range_kind == 1 && degree < 0) return fail(TBF_ERR_PARAM, "degree must be >= 0");
    const long long count = samples ? (long long)n : (long long)B * H * W;
    if (count <= 0) return fail(TBF_ERR_DIM, "no output pixels");
    const unsigned grid = (unsigned)std::min<long long>(count, 148LL * 16);
    k_bilateral_direct<T><<<grid, BF_THREADS, 0, (cudaStream_t)stream>>>(
        f, B, H, W, samples, count, taps, radius, range_kind, range_param, degree, out,
        d_counters ? d_counters + 1 : nullptr);
    return check_cuda("bilateral_direct");
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

extern "C" {

int32_t tbf_abi_version(void) { return TBF_ABI_VERSION; }

int tbf_profile_enable(int32_t on) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof_on = on != 0;
    return TBF_OK;
}

int32_t tbf_profile_kinds(void) { return KK_COUNT; }

int tbf_set_option(int32_t option, int64_t value) {
    switch (option) {
        case TBF_OPT_PIPELINE:
            g_pipeline = value != 0;
            return TBF_OK;
        case TBF_OPT_P1_YCHUNKS:
            if (value < 0 || value > TBF_MAX_YCH)
                return fail(TBF_ERR_PARAM, "pass-1 y-chunks must be in [0, %d]", TBF_MAX_YCH);
            g_p1_ychunks = (int)value;
            return TBF_OK;
        case TBF_OPT_P1_OCC:
            if (value < 2 || value > 3) return fail(TBF_ERR_PARAM, "pass-1 occupancy must be 2 or 3");
            g_p1_occ = (int)value;
            return TBF_OK;
        case TBF_OPT_P2_CHUNKS:
            g_p2_chunks = (int)std::max<int64_t>(0, value);
            return TBF_OK;
        case TBF_OPT_HOST_STRIPS:
            g_host_strips = (int)std::max<int64_t>(0, std::min<int64_t>(64, value));
            return TBF_OK;
        case TBF_OPT_HOST_BANDS:
            g_host_bands = (int)std::max<int64_t>(0, std::min<int64_t>(64, value));
            return TBF_OK;
        case TBF_OPT_P2_ORDER:
            g_p2_order = (int)std::max<int64_t>(0, std::min<int64_t>(3, value));
            return TBF_OK;
        case TBF_OPT_P1_FOLD:
            g_pass1_fold = value != 0;
            return TBF_OK;
        case TBF_OPT_LPT_SPLIT:
            g_lpt_split = (int)(value & 15);
            return TBF_OK;
        case TBF_OPT_P1_CLUSTER:
            if (value < 1 || value > 8) return fail(TBF_ERR_PARAM, "pass-1 cluster size must be in [1, 8]");
            g_p1_cluster = (int)value;
            return TBF_OK;
        case TBF_OPT_ZERO_UNIT:
            g_zero_unit = value != 0;
            return TBF_OK;
        case TBF_OPT_BATCHES:
            if (value < 1) return fail(TBF_ERR_PARAM, "batches must be >= 1");
            g_auto_batches = (int)value;
            return TBF_OK;
        default:
            return fail(TBF_ERR_PARAM, "unknown option %d", option);
    }
}

const char* tbf_kernel_name(int32_t kind) {
    return (kind >= 0 && kind < KK_COUNT) ? kKernelNames[kind] : "";
}

int32_t tbf_profile_timeline(double* start_ms, double* dur_ms, int32_t* kind, int32_t cap) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    int32_t n = 0;
    cudaEvent_t t0 = g_prof.empty() ? nullptr : g_prof.front().a;
    for (auto& r : g_prof) {
        float t = 0.f, s0 = 0.f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&t, r.a, r.b);
        cudaEventElapsedTime(&s0, t0, r.a);
        if (n < cap) {
            start_ms[n] = s0;
            dur_ms[n] = t;
            kind[n] = r.kind;
            ++n;
        }
    }
    for (auto& r : g_prof) {
        g_ev_pool.push_back(r.a);
        g_ev_pool.push_back(r.b);
    }
    g_prof.clear();
    return n;
}

int tbf_profile_collect(double* ms, long long* launches, int32_t n) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    for (int k = 0; k < n; ++k) {
        ms[k] = 0.0;
        launches[k] = 0;
    }
    int rc = TBF_OK;
    for (auto& r : g_prof) {
        float t = 0.f;
        if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess)
            rc = fail(TBF_ERR_CUDA, "profile event: %s", cudaGetErrorString(cudaGetLastError()));
        if (r.kind < n) {
            ms[r.kind] += t;
            launches[r.kind] += 1;
        }
        g_ev_pool.push_back(r.a);
        g_ev_pool.push_back(r.b);
    }
    g_prof.clear();
    return rc;
}

const char* tbf_last_error(void) { return g_last_error.c_str(); }

int tbf_layout_info(int32_t B, int32_t H, int32_t W, const tbf_spatial* sp, int32_t term_begin,
                    int32_t term_end, int32_t batch_terms, int32_t host_entry, int32_t* info, int32_t n_info) {
    if (!info || n_info < TBF_LAYOUT_INFO_N) return fail(TBF_ERR_PARAM, "info needs %d entries", TBF_LAYOUT_INFO_N);
    if (term_end <= term_begin) return fail(TBF_ERR_PARAM, "empty term range");
    Layout L;
    int rc = make_layout(B, H, W, sp, term_end - term_begin, batch_terms, &L, host_entry ? 0 : 1);
    if (rc) return rc;
    const bool box = sp->kind == TBF_SPATIAL_BOX;
    const int n = std::min(L.tb, term_end - term_begin);  // first batch
    const int npart = box ? -1 : (((n + G2 - 1) / G2 + P2R_GR - 1) / P2R_GR);
    const bool hpipe = host_entry && !box && L.nslot == 1;
    const P2Plan pp = p2_chunk_plan(L, sp, (n + G2 - 1) / G2, npart, hpipe);
    const int32_t v[TBF_LAYOUT_INFO_N] = {L.nb, L.tb, L.nyc, L.ych_lpt ? 1 : 0,
                                          L.nyc > 1 ? L.ychb[1] : H, L.nyc > 2 ? L.ychb[2] : H, L.ych_rows,
                                          pp.nchunk, pp.xlpt, pp.xlpt ? pp.xb1 : std::min(L.ntx, pp.tiles_per_chunk),
                                          pp.xlpt ? pp.xb2 : std::min(L.ntx, 2 * pp.tiles_per_chunk),
                                          pp.tiles_per_chunk, pp.xord, L.ntx};
    std::copy(v, v + TBF_LAYOUT_INFO_N, info);
    return TBF_OK;
}

size_t tbf_workspace_bytes(int32_t B, int32_t H, int32_t W, const tbf_spatial* sp,
                           int32_t term_begin, int32_t term_end, int32_t batch_terms) {
    // large enough for both the planned (device entry) and the equal-chunk
    // (host entry) layouts
    Layout L, Le;
    if (term_end <= term_begin) return 0;
    if (make_layout(B, H, W, sp, term_end - term_begin, batch_terms, &L, 2)) return 0;
    if (make_layout(B, H, W, sp, term_end - term_begin, batch_terms, &Le, 0)) return 0;
    return std::max(L.total, Le.total);
}

int tbf_range_check(const float* f, int64_t count, double T, unsigned long long* d_counters,
                    void* stream) {
    if (count <= 0) return fail(TBF_ERR_DIM, "empty input");
    if (!d_counters) return fail(TBF_ERR_PARAM, "null counters");
    cudaStream_t st = (cudaStream_t)stream;
    long long blocks = std::min<long long>((count + 255) / 256, 148LL * 8);
    { Prof pr(KK_RANGE, st); k_range_check<<<(unsigned)blocks, 256, 0, st>>>(f, count, -1e-9, T + 1e-9, d_counters); }
    return check_cuda("range_check");
}

int tbf_bilateral_trig(const float* f, float* out, int32_t B, int32_t H, int32_t W,
                       const tbf_spatial* sp, const tbf_terms* terms, int32_t batch_terms,
                       void* workspace, size_t workspace_bytes, unsigned long long* d_counters,
                       void* stream) {
    if (!terms) return fail(TBF_ERR_PARAM, "null terms");
    cudaStream_t st = (cudaStream_t)stream;
    // the range check runs inside run_terms (fused with the transpose)
    return run_terms(f, nullptr, nullptr, out, B, H, W, sp, terms, 0, terms->n_terms, batch_terms,
                     0, workspace, workspace_bytes, d_counters, st);
}

int tbf_bilateral_trig_host(const float* h_f, float* h_out, int32_t B, int32_t H, int32_t W,
                            const tbf_spatial* sp, const tbf_terms* terms, int32_t batch_terms,
                            float* d_io, void* workspace, size_t workspace_bytes,
                            unsigned long long* d_counters, void* stream) {
    if (!terms) return fail(TBF_ERR_PARAM, "null terms");
    if (!h_f || !h_out || !d_io) return fail(TBF_ERR_PARAM, "null host or device buffer");
    if (B < 1 || H < 1 || W < 1) return fail(TBF_ERR_DIM, "bad shape B=%d H=%d W=%d", B, H, W);
    // automatic split (same-box sweeps, scripts/host_sweep.py): images of
    // >= 8 MiB copy in column strips (pass 1 of a strip starts as it lands;
    // more than a few strips leave each launch under-filled while the x chain
    // serialises them) and return in row bands (the copy-back overlaps the
    // last pass 2).  Config 2 (16 MiB): 2 strips + 4 bands 1.87 ms per call,
    // 1 + 1 2.31 ms, 4 + 4 2.17 ms; config 5 (1 GiB): 4-8 strips and 8-24
    // bands within 0.5%, 2 strips +3%, 12 strips +2%.
    const int nrb = (H + P2_THREADS - 1) / P2_THREADS;
    const size_t bytes = (size_t)B * H * W * 4;
    const int strips = g_host_strips > 0 ? g_host_strips
                                         : (bytes < ((size_t)8 << 20) ? 1 : (bytes < ((size_t)128 << 20) ? 2 : 4));
    const int bands = g_host_bands > 0 ? g_host_bands : (nrb < 8 ? 1 : (bytes < ((size_t)128 << 20) ? 4 : 8));
    HostIO hio{h_f, h_out, strips, bands};
    float* d_f = d_io;
    float* d_out = d_io + (size_t)B * H * W;
    return run_terms(d_f, nullptr, nullptr, d_out, B, H, W, sp, terms, 0, terms->n_terms, batch_terms,
                     0, workspace, workspace_bytes, d_counters, (cudaStream_t)stream, &hio);
}

int tbf_trig_partial(const float* f, float* num, float* den, int32_t B, int32_t H, int32_t W,
                     const tbf_spatial* sp, const tbf_terms* terms, int32_t term_begin,
                     int32_t term_end, int32_t batch_terms, int32_t accumulate, void* workspace,
                     size_t workspace_bytes, void* stream) {
    if (!num || !den) return fail(TBF_ERR_PARAM, "null num/den");
    return run_terms(f, num, den, nullptr, B, H, W, sp, terms, term_begin, term_end, batch_terms,
                     accumulate, workspace, workspace_bytes, nullptr, (cudaStream_t)stream);
}

int tbf_trig_partial_rows(const float* f, float* num, float* den, int32_t B, int32_t H, int32_t W,
                          const tbf_spatial* sp, const tbf_terms* terms, int32_t term_begin, int32_t term_end,
                          int32_t row_begin, int32_t row_end, int32_t batch_terms, int32_t accumulate,
                          void* workspace, size_t workspace_bytes, void* stream) {
    if (!num || !den) return fail(TBF_ERR_PARAM, "null num/den");
    return run_terms(f, num, den, nullptr, B, H, W, sp, terms, term_begin, term_end, batch_terms, accumulate,
                     workspace, workspace_bytes, nullptr, (cudaStream_t)stream, nullptr, row_begin, row_end);
}

int tbf_finalize(const float* num, const float* den, const float* f, float* out, int64_t count,
                 unsigned long long* d_counters, void* stream) {
    if (count <= 0) return fail(TBF_ERR_DIM, "empty input");
    long long blocks = std::min<long long>((count + 255) / 256, 148LL * 8);
    {
        Prof pr(KK_FINALIZE, (cudaStream_t)stream);
        k_finalize<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(num, den, f, out, count,
                                                                       d_counters);
    }
    return check_cuda("finalize");
}

int tbf_recursive_smooth_f64(const double* a, double* out, int32_t h, int32_t w, double scale,
                             double c1, double c2, double c3, double c4, int32_t pad,
                             double* scratch, void* stream) {
    if (h < 1 || w < 1) return fail(TBF_ERR_DIM, "bad shape %dx%d", h, w);
    if (pad < 0) return fail(TBF_ERR_PARAM, "pad must be >= 0");
    k_recursive_smooth_f64<<<(w + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
        a, out, h, w, scale, c1, c2, c3, c4, pad, scratch);
    return check_cuda("recursive_smooth_f64");
}


int tbf_bilateral_direct(const float* f, int32_t B, int32_t H, int32_t W, const int32_t* samples,
                         int64_t n, const double* taps, int32_t radius, int32_t range_kind,
                         double range_param, int32_t degree, double* out, unsigned long long* d_counters,
                         void* stream) {
    return bilateral_direct_impl(f, B, H, W, samples, n, taps, radius, range_kind, range_param, degree, out,
                                 d_counters, stream);
}

int tbf_bilateral_direct_f64(const double* f, int32_t B, int32_t H, int32_t W, const int32_t* samples,
                             int64_t n, const double* taps, int32_t radius, int32_t range_kind,
                             double range_param, int32_t degree, double* out, unsigned long long* d_counters,
                             void* stream) {
    return bilateral_direct_impl(f, B, H, W, samples, n, taps, radius, range_kind, range_param, degree, out,
                                 d_counters, stream);
}

int tbf_box_pass_f64(const double* a, double* out, int32_t h, int32_t w, int32_t radius,
                     void* stream) {
    if (h < 1 || w < 1) return fail(TBF_ERR_DIM, "bad shape %dx%d", h, w);
    if (radius < 0) return fail(TBF_ERR_PARAM, "box radius must be >= 0, got %d", radius);
    k_box_pass_f64<<<(h + 127) / 128, 128, 0, (cudaStream_t)stream>>>(a, out, h, w, radius);
    return check_cuda("box_pass_f64");
}

}  // extern "C"
