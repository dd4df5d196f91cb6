// flowmdp_b200.cu -- B200 (sm_100a) kernels + C ABI for the planner hot path
// of arXiv 2109.00857: ensemble-counted MDP model build and backward
// Bellman solve.  See DESIGN.md for the data layout and roofline, and
// include/flowmdp_b200.h for the reference function each entry replaces.
//
// Exactness contract: all position / reward / value
// arithmetic is f64 with explicitly rounded __dadd_rn/__dmul_rn/__ddiv_rn
// (and the file is compiled with -fmad=false), reproducing the numpy
// reference's operation order so counts, columns, probabilities, rewards,
// values and the policy are bit-identical.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <cfloat>
#include <climits>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/flowmdp_b200.h"
#include "fm_hypot.cuh"

#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))
#define DMUL(a, b) __dmul_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))

static constexpr unsigned kFull = 0xffffffffu;

// realizations per reconstruction chunk of k_build
#ifndef FM_BUILD_RC
#define FM_BUILD_RC 64
#endif

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

static int32_t fm_fail(int32_t code, const char *fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define FM_CK(expr)                                                                     \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fm_fail(FM_CUDA_ERROR, "%s failed: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

static std::atomic<long long> g_launches{0};

// every kernel launch site reports through here (fm_kernel_launches)
#define FM_CK_LAUNCH_N(name, n)                                                         \
    do {                                                                                \
        g_launches += (n);                                                              \
        cudaError_t e_ = cudaGetLastError();                                            \
        if (e_ != cudaSuccess)                                                          \
            return fm_fail(FM_CUDA_ERROR, "launch %s: %s", name, cudaGetErrorString(e_)); \
    } while (0)

#define FM_CK_LAUNCH(name)                                                              \
    do {                                                                                \
        g_launches += 1;                                                                \
        cudaError_t e_ = cudaGetLastError();                                            \
        if (e_ != cudaSuccess)                                                          \
            return fm_fail(FM_CUDA_ERROR, "launch %s: %s", name, cudaGetErrorString(e_)); \
    } while (0)

extern "C" int32_t fm_abi_version(void) { return 1; }
extern "C" const char *fm_last_error(void) { return g_err.c_str(); }
extern "C" int64_t fm_kernel_launches(void) { return g_launches.load(); }

static int sm_count()
{
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Development counters (-DFM_STATS): [0] rare transitions, [1] exact
// segment samplings, [2] segment samples, [3] transitions in obstacle warps,
// [4] transitions in lean warps (per transition), [5] binned tasks, [6]
// realizations of binned tasks taking the exact path, [7] lean tasks of a
// bin launch that did not fit the bins.  Not part of the ABI header.
#ifdef FM_STATS
__device__ unsigned long long g_fm_stats[8];
#define FM_STAT(i, n) atomicAdd(&g_fm_stats[i], (unsigned long long)(n))
// per-task cycle counts of PART-2 launches (dev: task id << 40 | path << 36 | cycles)
__device__ unsigned long long g_fm_ttimes[1 << 20];
__device__ unsigned int g_fm_tcount;
// per-warp counters of the current task (dev): [warp][0] D items, [1] gated items, [2] pairs, [3] seg tests
__device__ unsigned int g_fm_wcnt[148 * 64][8];   // + [4] init cycles/64, [5] drain cycles/64, [6] loop+drain cycles/64
#else
#define FM_STAT(i, n) ((void)0)
#endif
extern "C" int32_t fm_dev_task_times(uint64_t *h_out, int32_t max_n, int32_t *h_n)
{
#ifdef FM_STATS
    unsigned int n = 0;
    FM_CK(cudaMemcpyFromSymbol(&n, g_fm_tcount, 4));
    if (n > (unsigned)max_n) n = (unsigned)max_n;
    if (n > (1u << 17)) n = 1u << 17;
    FM_CK(cudaMemcpyFromSymbol(h_out, g_fm_ttimes, 8ull << 20));
    *h_n = (int32_t)n;
    const unsigned int z = 0;
    FM_CK(cudaMemcpyToSymbol(g_fm_tcount, &z, 4));
    return FM_OK;
#else
    (void)h_out; (void)max_n;
    *h_n = 0;
    return FM_OK;
#endif
}
extern "C" int32_t fm_dev_stats(uint64_t *h_out8)
{
#ifdef FM_STATS
    FM_CK(cudaMemcpyFromSymbol(h_out8, g_fm_stats, 64));
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    FM_CK(cudaMemcpyToSymbol(g_fm_stats, z, 64));
#else
    for (int i = 0; i < 8; ++i) h_out8[i] = 0;
#endif
    return FM_OK;
}

// Keep the stream-ordered pool's memory across synchronisations (the
// default release threshold of 0 hands it back at every sync, so the next
// cudaMallocAsync of a planner step would map fresh pages).
static void pool_keep()
{
    static bool done = false;
    if (done) return;
    done = true;
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
}

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
// max that keeps a NaN (numpy's max propagates it)
__device__ __forceinline__ double nan_max(double m, double x) { return (x != x || x > m) ? x : m; }

__device__ __forceinline__ double warp_max_f64(double v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v = nan_max(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// non-negative doubles order like their bit patterns
__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v)
{
    atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}

// ---------------------------------------------------------------------------
// K_vmax: compute_subgrid's exact scan (model_builder.py:392-396)
//
// max over (t, r, cell) of |v_x| and |v_y|, exact.  The scan runs in FP32
// (FFMA, smem-staged coefficients) with a rigorous per-cell error bound
//   |v32 - v| <= delta = (2 n_m + 8) 2^-24 T + tiny,
//   T = |mean| + sum_m |mode_m| max_r |coeff_{t,r,m}|   (>= every partial sum),
// and only elements with |v32| >= rd(E - delta), E the running exact max,
// are recomputed in f64 with the reference's operation order.  The true
// maximiser always passes that test, so the result is the exact f64 max;
// recomputes happen O(log N_rv) times per cell.
// ---------------------------------------------------------------------------
static constexpr int kVmaxChunk = 64;

template <int NMX>
__device__ __noinline__ double vmax_exact_component(const fm_grid G, const fm_env E, int t, int r, int c, int comp)
{
    const int nc = G.nx * G.ny;
    double v = E.mean[((size_t)t * nc + c) * 2 + comp];
    const double *cf = E.coeffs + ((size_t)t * E.n_real + r) * E.n_modes;
    for (int m = 0; m < E.n_modes; ++m)
        v = DADD(v, DMUL(cf[m], E.modes[(((size_t)m * G.nt + t) * nc + c) * 2 + comp]));
    return fabs(v);
}

// packed 2 x FP32 fused multiply-add (sm_100 FFMA2): a * (b.x, b.y) + c
__device__ __forceinline__ float2 ffma2_bcast(float a, float2 b, float2 c)
{
    unsigned long long r;
    const float2 aa = make_float2(a, a);
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const unsigned long long *>(&aa)),
          "l"(*reinterpret_cast<const unsigned long long *>(&b)),
          "l"(*reinterpret_cast<const unsigned long long *>(&c)));
    return *reinterpret_cast<float2 *>(&r);
}

// Each thread scans two cells (c, c + 256) so every staged coefficient feeds
// two FFMA2 chains; the running exact maxima are shared by the two cells
// (an element can only raise the global maximum if |v32| >= E - delta_cell).
static constexpr int kVmaxCells = 2;
#ifndef FM_VMAX_STEP
#define FM_VMAX_STEP 4
#endif
static constexpr int kVmaxStep = FM_VMAX_STEP;   // realizations per step

// Per-(t, cell) velocity envelope (the build's bin ranges): int4 of
// order-preserving encodings of f32 (x_lo, x_hi, y_lo, y_hi), each already
// widened by the cell's error bound so it contains every exact f64 value.
__device__ __forceinline__ int f32_ord(float f)
{
    const int b = __float_as_int(f);
    return b >= 0 ? b : b ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float ord_f32(int e) { return __int_as_float(e >= 0 ? e : e ^ 0x7FFFFFFF); }

__device__ __forceinline__ void store_envelope(int4 *vr, size_t idx, float xlo, float xhi, float ylo, float yhi,
                                               bool direct)
{
    const int4 e = make_int4(f32_ord(xlo), f32_ord(xhi), f32_ord(ylo), f32_ord(yhi));
    if (direct) {
        vr[idx] = e;
    } else {
        int *p = reinterpret_cast<int *>(vr + idx);
        atomicMin(p, e.x);
        atomicMax(p + 1, e.y);
        atomicMin(p + 2, e.z);
        atomicMax(p + 3, e.w);
    }
}

__global__ void k_envelope_init(int4 *vr, int nc, int t0, int nts, int cell0, int ncell)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)nts * ncell) return;
    const int t = t0 + (int)(i / ncell), c = cell0 + (int)(i % ncell);
    const int pinf = 0x7f800000, ninf = f32_ord(__int_as_float(0xff800000));
    vr[(size_t)t * nc + c] = make_int4(pinf, ninf, pinf, ninf);
}

// EXACT: the exact maxima (out2[0..1]); otherwise bounds only (out2[0..3] =
// lo_x, hi_x, lo_y, hi_y with lo <= max|v_c| <= hi, from the f32 envelope
// widened by the per-cell error bound; +inf if an input is not finite) and
// the envelope -- no per-element threshold test, no f64 recompute.
template <int NMX, bool EXACT = true>
__global__ void __launch_bounds__(256) k_vmax(fm_grid G, fm_env E, int t0, int cell0, int ncell, int r_per_block,
                                               const double *cmax, double *out2, int4 *vrange)
{
    __shared__ float cs[kVmaxChunk][NMX];
    const int nc = G.nx * G.ny;
    const int t = t0 + blockIdx.y;   // cmax holds the slab's layers only
    const int nm = E.n_modes;
    const int r_lo = blockIdx.z * r_per_block;
    const int r_hi = min(E.n_real, r_lo + r_per_block);
    int cell[kVmaxCells];
    bool ok[kVmaxCells];
    float2 mu32[kVmaxCells];
    float2 d32[kVmaxCells][NMX];
    double delx[kVmaxCells], dely[kVmaxCells];
#pragma unroll
    for (int q = 0; q < kVmaxCells; ++q) {
        const int lc = blockIdx.x * blockDim.x * kVmaxCells + q * blockDim.x + threadIdx.x;
        const int c = cell0 + lc;   // cells of the row strip [cell0, cell0 + ncell)
        cell[q] = c;
        ok[q] = lc < ncell;
        mu32[q] = make_float2(0.f, 0.f);
        double Tx = 0.0, Ty = 0.0;
#pragma unroll
        for (int m = 0; m < NMX; ++m) d32[q][m] = make_float2(0.f, 0.f);
        if (ok[q]) {
            const double2 mu = *reinterpret_cast<const double2 *>(E.mean + ((size_t)t * nc + c) * 2);
            mu32[q] = make_float2((float)mu.x, (float)mu.y);
            Tx = fabs(mu.x);
            Ty = fabs(mu.y);
#pragma unroll
            for (int m = 0; m < NMX; ++m) {
                if (m < nm) {
                    const double2 md =
                        *reinterpret_cast<const double2 *>(E.modes + (((size_t)m * G.nt + t) * nc + c) * 2);
                    d32[q][m] = make_float2((float)md.x, (float)md.y);
                    const double cm = cmax[(size_t)(t - t0) * nm + m];
                    Tx += fabs(md.x) * cm;
                    Ty += fabs(md.y) * cm;
                }
            }
        }
        const double kRel = (2.0 * nm + 8.0) * 0x1p-24 * 1.001, kAbs = (nm + 2.0) * 0x1p-140;
        delx[q] = Tx * kRel + kAbs;
        dely[q] = Ty * kRel + kAbs;
    }
    double ex = 0.0, ey = 0.0;   // running exact maxima (shared by this thread's cells)
    float2 vlo[kVmaxCells], vhi[kVmaxCells];   // envelope of the f32 reconstructions
#pragma unroll
    for (int q = 0; q < kVmaxCells; ++q) {
        vlo[q] = make_float2(__int_as_float(0x7f800000), __int_as_float(0x7f800000));
        vhi[q] = make_float2(__int_as_float(0xff800000), __int_as_float(0xff800000));
    }
    float thx[kVmaxCells], thy[kVmaxCells];
#pragma unroll
    for (int q = 0; q < kVmaxCells; ++q) {
        // a cell past the grid never passes: its threshold is +inf
        thx[q] = ok[q] ? __double2float_rd(-delx[q]) : __int_as_float(0x7f800000);
        thy[q] = ok[q] ? __double2float_rd(-dely[q]) : __int_as_float(0x7f800000);
    }
    for (int r0 = r_lo; r0 < r_hi; r0 += kVmaxChunk) {
        const int n = min(kVmaxChunk, r_hi - r0);
        __syncthreads();
        for (int i = threadIdx.x; i < n * NMX; i += blockDim.x) {
            const int k = i / NMX, m = i % NMX;
            cs[k][m] = m < nm ? (float)E.coeffs[((size_t)t * E.n_real + r0 + k) * nm + m] : 0.f;
        }
        __syncthreads();
        if (!ok[0]) continue;
        // kVmaxStep realizations per step; (vx, vy) in one packed FFMA2 chain.
        // Unused modes hold zeros (exact no-ops), so no mode-count test.
        // A step past the chunk's end re-evaluates its last realization
        // (harmless for a maximum).
        for (int k = 0; k < n; k += kVmaxStep) {
            int kk[kVmaxStep];
#pragma unroll
            for (int j = 0; j < kVmaxStep; ++j) kk[j] = min(k + j, n - 1);
            float2 v[kVmaxStep][kVmaxCells];
#pragma unroll
            for (int j = 0; j < kVmaxStep; ++j)
#pragma unroll
                for (int q = 0; q < kVmaxCells; ++q) v[j][q] = mu32[q];
#pragma unroll
            for (int m = 0; m < NMX; ++m) {
#pragma unroll
                for (int j = 0; j < kVmaxStep; ++j) {
                    const float cj = cs[kk[j]][m];
#pragma unroll
                    for (int q = 0; q < kVmaxCells; ++q) v[j][q] = ffma2_bcast(cj, d32[q][m], v[j][q]);
                }
            }
            if (vrange || !EXACT) {
#pragma unroll
                for (int j = 0; j < kVmaxStep; ++j)
#pragma unroll
                    for (int q = 0; q < kVmaxCells; ++q) {
                        vlo[q].x = fminf(vlo[q].x, v[j][q].x);
                        vhi[q].x = fmaxf(vhi[q].x, v[j][q].x);
                        vlo[q].y = fminf(vlo[q].y, v[j][q].y);
                        vhi[q].y = fmaxf(vhi[q].y, v[j][q].y);
                    }
            }
            if (!EXACT) continue;
            // !(|v| < th) also routes NaN / inf to the exact path
            bool hit = false;
#pragma unroll
            for (int j = 0; j < kVmaxStep; ++j)
#pragma unroll
                for (int q = 0; q < kVmaxCells; ++q)
                    hit = hit || !(fabsf(v[j][q].x) < thx[q]) || !(fabsf(v[j][q].y) < thy[q]);
            if (hit) {
#pragma unroll
                for (int q = 0; q < kVmaxCells; ++q) {
#pragma unroll
                    for (int j = 0; j < kVmaxStep; ++j) {
                        const float2 vv = v[j][q];
                        const int r = r0 + kk[j];
                        if (!(fabsf(vv.x) < thx[q])) {
                            const double e = vmax_exact_component<NMX>(G, E, t, r, cell[q], 0);
                            ex = (e != e || e > ex) ? e : ex;   // NaN sticks (the reference's max propagates it)
#pragma unroll
                            for (int qq = 0; qq < kVmaxCells; ++qq)
                                if (ok[qq]) thx[qq] = __double2float_rd(ex - delx[qq]);
                        }
                        if (!(fabsf(vv.y) < thy[q])) {
                            const double e = vmax_exact_component<NMX>(G, E, t, r, cell[q], 1);
                            ey = (e != e || e > ey) ? e : ey;
#pragma unroll
                            for (int qq = 0; qq < kVmaxCells; ++qq)
                                if (ok[qq]) thy[qq] = __double2float_rd(ey - dely[qq]);
                        }
                    }
                }
            }
        }
    }
    if (vrange) {
        // widened by the cell's bound delta >= |v32 - v64| (rounded outwards)
#pragma unroll
        for (int q = 0; q < kVmaxCells; ++q)
            if (ok[q])
                store_envelope(vrange, (size_t)t * nc + cell[q], __fsub_rd(vlo[q].x, __double2float_ru(delx[q])),
                               __fadd_ru(vhi[q].x, __double2float_ru(delx[q])),
                               __fsub_rd(vlo[q].y, __double2float_ru(dely[q])),
                               __fadd_ru(vhi[q].y, __double2float_ru(dely[q])), gridDim.z == 1);
    }
    if constexpr (!EXACT) {
        double lox = 0.0, hix = 0.0, loy = 0.0, hiy = 0.0;
#pragma unroll
        for (int q = 0; q < kVmaxCells; ++q) {
            if (!ok[q]) continue;
            const double ax = fmax(-(double)vlo[q].x, (double)vhi[q].x), ay = fmax(-(double)vlo[q].y, (double)vhi[q].y);
            // a non-finite input (or a bound that is not small) -> +inf: the caller takes the exact scan
            const bool fin = delx[q] < 1e30 && dely[q] < 1e30;
            lox = fmax(lox, __dsub_rd(ax, delx[q]));
            hix = fin ? fmax(hix, __dadd_ru(ax, delx[q])) : __longlong_as_double(0x7ff0000000000000LL);
            loy = fmax(loy, __dsub_rd(ay, dely[q]));
            hiy = fin ? fmax(hiy, __dadd_ru(ay, dely[q])) : __longlong_as_double(0x7ff0000000000000LL);
        }
        lox = warp_max_f64(lox);
        hix = warp_max_f64(hix);
        loy = warp_max_f64(loy);
        hiy = warp_max_f64(hiy);
        if ((threadIdx.x & 31) == 0) {
            atomic_max_nonneg(out2, lox);
            atomic_max_nonneg(out2 + 1, hix);
            atomic_max_nonneg(out2 + 2, loy);
            atomic_max_nonneg(out2 + 3, hiy);
        }
        return;
    }
    // non-negative doubles (and +NaN, above +inf) order like their bit patterns
    unsigned long long bx = (unsigned long long)__double_as_longlong(ex),
                       by = (unsigned long long)__double_as_longlong(ey);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long ox = __shfl_xor_sync(kFull, bx, o), oy = __shfl_xor_sync(kFull, by, o);
        bx = ox > bx ? ox : bx;
        by = oy > by ? oy : by;
    }
    ex = __longlong_as_double((long long)bx);
    ey = __longlong_as_double((long long)by);
    if ((threadIdx.x & 31) == 0) {
        atomic_max_nonneg(out2, ex);
        atomic_max_nonneg(out2 + 1, ey);
    }
}

__global__ void k_maxabs_seg(const double *src, int64_t seg_len, int64_t elem_stride, int64_t inner,
                             int64_t outer_stride, int64_t inner_stride, double *out);

// ---------------------------------------------------------------------------
// k_vmax_tc: the bounds-only envelope scan (k_vmax<8, false>) with the
// coefficient x mode contraction on the tensor cores (north_star: "tensor
// cores for that contraction only if it holds tolerance").  Per warp and
// step: 16 realizations x 4 cells x (vx, vy) = one m16n8k8 TF32 MMA tile
// (A = coefficients [realization][mode], B = modes [mode][cell, component],
// C = mean), run as 3xTF32 (A_lo B_hi + A_hi B_lo + A_hi B_hi: the
// operands split into two TF32 halves, 2^-22 relative each) so the result
// carries ~f32 accuracy.  The envelope and the bounds only need a rigorous
// outer bound, never the f32 value itself: |v_tc - v64| <= delta_tc =
// 2^-16 T + abs, T = |mean| + sum_m |mode_m| max_r |coeff_m| -- the split
// (3 * 2^-22 per product) and up to 64 ulps of f32 accumulation error
// (truncating adds included) are < 2^-17 T, so the factor 2 is slack.
// (The build's bins only need the envelope as a box hint: a realization
// outside it takes the exact path, bin_setup.)  Lanes: g = lane >> 2 (row
// of the tile: realizations g, g + 8), q = lane & 3 (the tile's cell, and
// the modes q, q + 4 of the A / B fragments).  Environment.py:293-297
// (reconstruction), model_builder.py:376-399 (the maxima it bounds).
// ---------------------------------------------------------------------------
static constexpr int kTcQuads = 2;      // 4-cell tiles per warp (independent MMA chains)
static constexpr int kTcChunk = 64;     // realizations staged per block step (4 MMA steps)

__device__ __forceinline__ unsigned tf32_rna(float x)
{
    unsigned r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1)
{
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(256) k_vmax_tc(fm_grid G, fm_env E, int t0, int cell0, int ncell, int r_per_block,
                                                 const double *cmax, double *out4, int4 *vrange)
{
    // [step][lane] fragments: (a0, a1, a2, a3) hi, then lo
    __shared__ uint4 cs_hi[kTcChunk / 16][32], cs_lo[kTcChunk / 16][32];
    const int nc = G.nx * G.ny, nm = E.n_modes;
    const int t = t0 + blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
    const int r_lo = blockIdx.z * r_per_block, r_hi = min(E.n_real, r_lo + r_per_block);
    // this lane's tile column (cell, component) for B, and its D cell
    unsigned bh0[kTcQuads], bh1[kTcQuads], bl0[kTcQuads], bl1[kTcQuads];
    float mux[kTcQuads], muy[kTcQuads];
    float2 vlo[kTcQuads], vhi[kTcQuads];
    int cell[kTcQuads];
    bool ok[kTcQuads];
    double dx_[kTcQuads], dy_[kTcQuads];
#pragma unroll
    for (int u = 0; u < kTcQuads; ++u) {
        const int tile = (blockIdx.x * (blockDim.x >> 5) + warp) * kTcQuads + u;
        // B column n = g: cell 4 tile + (g >> 1), component g & 1
        const int lb = tile * 4 + (g >> 1), cb = cell0 + lb;
        float m0 = 0.f, m1 = 0.f;
        if (lb < ncell) {
            if (q < nm) m0 = (float)E.modes[(((size_t)q * G.nt + t) * nc + cb) * 2 + (g & 1)];
            if (q + 4 < nm) m1 = (float)E.modes[(((size_t)(q + 4) * G.nt + t) * nc + cb) * 2 + (g & 1)];
        }
        bh0[u] = tf32_rna(m0);
        bh1[u] = tf32_rna(m1);
        bl0[u] = tf32_rna(m0 - __uint_as_float(bh0[u]));
        bl1[u] = tf32_rna(m1 - __uint_as_float(bh1[u]));
        // D cell: 4 tile + q
        const int ld = tile * 4 + q, cd = cell0 + ld;
        ok[u] = ld < ncell;
        cell[u] = cd;
        mux[u] = muy[u] = 0.f;
        double Tx = 0.0, Ty = 0.0;
        if (ok[u]) {
            const double2 mu = *reinterpret_cast<const double2 *>(E.mean + ((size_t)t * nc + cd) * 2);
            mux[u] = (float)mu.x;
            muy[u] = (float)mu.y;
            Tx = fabs(mu.x);
            Ty = fabs(mu.y);
            for (int m = 0; m < nm; ++m) {
                const double2 md = *reinterpret_cast<const double2 *>(E.modes + (((size_t)m * G.nt + t) * nc + cd) * 2);
                const double cm = cmax[(size_t)(t - t0) * nm + m];
                Tx += fabs(md.x) * cm;
                Ty += fabs(md.y) * cm;
            }
        }
        const double kRel = 0x1p-16, kAbs = (nm + 2.0) * 0x1p-140;
        dx_[u] = Tx * kRel + kAbs;
        dy_[u] = Ty * kRel + kAbs;
        vlo[u] = make_float2(__int_as_float(0x7f800000), __int_as_float(0x7f800000));
        vhi[u] = make_float2(__int_as_float(0xff800000), __int_as_float(0xff800000));
    }
    for (int r0 = r_lo; r0 < r_hi; r0 += kTcChunk) {
        const int n = min(kTcChunk, r_hi - r0);
        __syncthreads();
        // stage the chunk as split TF32 fragments (a realization past the
        // end repeats the last one: harmless for a min / max)
        for (int i = threadIdx.x; i < kTcChunk * 8; i += blockDim.x) {
            const int k = i >> 3, m = i & 7;
            const int kk = min(k, n - 1);
            const float c = m < nm ? (float)E.coeffs[((size_t)t * E.n_real + r0 + kk) * nm + m] : 0.f;
            const unsigned h = tf32_rna(c), l = tf32_rna(c - __uint_as_float(h));
            const int st = k >> 4, rl = k & 15;
            const int ln = (rl & 7) * 4 + (m & 3), sl = (rl >> 3) + 2 * (m >> 2);
            reinterpret_cast<unsigned *>(&cs_hi[st][ln])[sl] = h;
            reinterpret_cast<unsigned *>(&cs_lo[st][ln])[sl] = l;
        }
        __syncthreads();
        for (int st = 0; st < (n + 15) >> 4; ++st) {
            const uint4 H = cs_hi[st][lane], L = cs_lo[st][lane];
            const unsigned ah[4] = {H.x, H.y, H.z, H.w}, al[4] = {L.x, L.y, L.z, L.w};
#pragma unroll
            for (int u = 0; u < kTcQuads; ++u) {
                float d[4] = {mux[u], muy[u], mux[u], muy[u]};
                mma_tf32(d, al, bh0[u], bh1[u]);
                mma_tf32(d, ah, bl0[u], bl1[u]);
                mma_tf32(d, ah, bh0[u], bh1[u]);
                vlo[u].x = fminf(vlo[u].x, fminf(d[0], d[2]));
                vhi[u].x = fmaxf(vhi[u].x, fmaxf(d[0], d[2]));
                vlo[u].y = fminf(vlo[u].y, fminf(d[1], d[3]));
                vhi[u].y = fmaxf(vhi[u].y, fmaxf(d[1], d[3]));
            }
        }
    }
    double lox = 0.0, hix = 0.0, loy = 0.0, hiy = 0.0;
#pragma unroll
    for (int u = 0; u < kTcQuads; ++u) {
        // the tile's rows: lanes with the same q (xor over the g bits)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            vlo[u].x = fminf(vlo[u].x, __shfl_xor_sync(kFull, vlo[u].x, o));
            vhi[u].x = fmaxf(vhi[u].x, __shfl_xor_sync(kFull, vhi[u].x, o));
            vlo[u].y = fminf(vlo[u].y, __shfl_xor_sync(kFull, vlo[u].y, o));
            vhi[u].y = fmaxf(vhi[u].y, __shfl_xor_sync(kFull, vhi[u].y, o));
        }
        if (g == 0 && ok[u]) {
            if (vrange)
                store_envelope(vrange, (size_t)t * nc + cell[u], __fsub_rd(vlo[u].x, __double2float_ru(dx_[u])),
                               __fadd_ru(vhi[u].x, __double2float_ru(dx_[u])),
                               __fsub_rd(vlo[u].y, __double2float_ru(dy_[u])),
                               __fadd_ru(vhi[u].y, __double2float_ru(dy_[u])), gridDim.z == 1);
            const double ax = fmax(-(double)vlo[u].x, (double)vhi[u].x), ay = fmax(-(double)vlo[u].y, (double)vhi[u].y);
            // a non-finite input (or a bound that is not small) -> +inf: the caller takes the exact scan
            const bool fin = dx_[u] < 1e30 && dy_[u] < 1e30;
            lox = fmax(lox, __dsub_rd(ax, dx_[u]));
            hix = fin ? fmax(hix, __dadd_ru(ax, dx_[u])) : __longlong_as_double(0x7ff0000000000000LL);
            loy = fmax(loy, __dsub_rd(ay, dy_[u]));
            hiy = fin ? fmax(hiy, __dadd_ru(ay, dy_[u])) : __longlong_as_double(0x7ff0000000000000LL);
        }
    }
    lox = warp_max_f64(lox);
    hix = warp_max_f64(hix);
    loy = warp_max_f64(loy);
    hiy = warp_max_f64(hiy);
    if (lane == 0) {
        atomic_max_nonneg(out4, lox);
        atomic_max_nonneg(out4 + 1, hix);
        atomic_max_nonneg(out4 + 2, loy);
        atomic_max_nonneg(out4 + 3, hiy);
    }
}


// More than 16 modes: the plain f64 scan (the filter's per-cell mode
// registers would not fit).  One thread per cell, RB realizations at a time,
// modes outer so each mode is loaded once per block of realizations; every
// realization's sum still runs in mode order (environment.py:293-297).
template <int RB>
__global__ void __launch_bounds__(256) k_vmax_f64(fm_grid G, fm_env E, int t0, int cell0, int ncell,
                                                   int r_per_block, double *out2, int4 *vrange)
{
    const int nc = G.nx * G.ny;
    const int t = t0 + blockIdx.y;
    const int nm = E.n_modes;
    const int lc = blockIdx.x * blockDim.x + threadIdx.x;
    const bool ok = lc < ncell;
    const int c = cell0 + (ok ? lc : 0);
    const int r_lo = blockIdx.z * r_per_block;
    const int r_hi = min(E.n_real, r_lo + r_per_block);
    double ex = 0.0, ey = 0.0;
    double lx = INFINITY, hx = -INFINITY, ly = INFINITY, hy = -INFINITY;   // exact envelope
    if (ok) {
        const double2 mu = *reinterpret_cast<const double2 *>(E.mean + ((size_t)t * nc + c) * 2);
        for (int r0 = r_lo; r0 < r_hi; r0 += RB) {
            double vx[RB], vy[RB];
#pragma unroll
            for (int q = 0; q < RB; ++q) vx[q] = mu.x, vy[q] = mu.y;
            for (int m = 0; m < nm; ++m) {
                const double2 md = *reinterpret_cast<const double2 *>(E.modes + (((size_t)m * G.nt + t) * nc + c) * 2);
#pragma unroll
                for (int q = 0; q < RB; ++q) {
                    const int r = min(r0 + q, r_hi - 1);   // past the end: a repeat, harmless for a max
                    const double cf = __ldg(E.coeffs + ((size_t)t * E.n_real + r) * nm + m);
                    vx[q] = DADD(vx[q], DMUL(cf, md.x));
                    vy[q] = DADD(vy[q], DMUL(cf, md.y));
                }
            }
#pragma unroll
            for (int q = 0; q < RB; ++q) {
                const double ax = fabs(vx[q]), ay = fabs(vy[q]);
                ex = (ax != ax || ax > ex) ? ax : ex;   // NaN sticks
                ey = (ay != ay || ay > ey) ? ay : ey;
                lx = fmin(lx, vx[q]);
                hx = fmax(hx, vx[q]);
                ly = fmin(ly, vy[q]);
                hy = fmax(hy, vy[q]);
            }
        }
        if (vrange)
            store_envelope(vrange, (size_t)t * nc + c, __double2float_rd(lx), __double2float_ru(hx),
                           __double2float_rd(ly), __double2float_ru(hy), gridDim.z == 1);
    }
    unsigned long long bx = (unsigned long long)__double_as_longlong(ex),
                       by = (unsigned long long)__double_as_longlong(ey);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long ox = __shfl_xor_sync(kFull, bx, o), oy = __shfl_xor_sync(kFull, by, o);
        bx = ox > bx ? ox : bx;
        by = oy > by ? oy : by;
    }
    if ((threadIdx.x & 31) == 0) {
        atomic_max_nonneg(out2, __longlong_as_double((long long)bx));
        atomic_max_nonneg(out2 + 1, __longlong_as_double((long long)by));
    }
}

extern "C" int32_t fm_velocity_max(fm_grid G, fm_env E, double *d_out2, void *stream)
{
    return fm_velocity_max_rows(G, E, 0, G.ny, d_out2, stream);
}

extern "C" int32_t fm_velocity_scan(fm_grid G, fm_env E, int32_t t0, int32_t t1, int32_t j0, int32_t j1,
                                    double *d_out2, int32_t *d_envelope, void *stream);

extern "C" int32_t fm_velocity_max_slab(fm_grid G, fm_env E, int32_t t0, int32_t t1, int32_t j0, int32_t j1,
                                        double *d_out2, void *stream)
{
    return fm_velocity_scan(G, E, t0, t1, j0, j1, d_out2, nullptr, stream);
}

extern "C" int32_t fm_velocity_max_rows(fm_grid G, fm_env E, int32_t j0, int32_t j1, double *d_out2, void *stream)
{
    return fm_velocity_max_slab(G, E, 0, G.nt, j0, j1, d_out2, stream);
}

static int32_t velocity_scan(fm_grid G, fm_env E, int32_t t0, int32_t t1, int32_t j0, int32_t j1, double *d_out2,
                             int32_t *d_envelope, void *stream, bool exact);

extern "C" int32_t fm_velocity_scan(fm_grid G, fm_env E, int32_t t0, int32_t t1, int32_t j0, int32_t j1,
                                    double *d_out2, int32_t *d_envelope, void *stream)
{
    return velocity_scan(G, E, t0, t1, j0, j1, d_out2, d_envelope, stream, true);
}

extern "C" int32_t fm_velocity_bounds(fm_grid G, fm_env E, int32_t t0, int32_t t1, int32_t j0, int32_t j1,
                                      double *d_out4, int32_t *d_envelope, void *stream)
{
    if (E.n_modes > 16) {   // the f64 scan (no f32 envelope): exact maxima as both bounds
        double *tmp = nullptr;
        cudaStream_t s = (cudaStream_t)stream;
        FM_CK(cudaMallocAsync(&tmp, 2 * sizeof(double), s));
        FM_CK(cudaMemsetAsync(tmp, 0, 2 * sizeof(double), s));
        const int32_t st = velocity_scan(G, E, t0, t1, j0, j1, tmp, d_envelope, stream, true);
        if (st != FM_OK) return st;
        for (int k = 0; k < 4; ++k)
            FM_CK(cudaMemcpyAsync(d_out4 + k, tmp + k / 2, sizeof(double), cudaMemcpyDeviceToDevice, s));
        FM_CK(cudaFreeAsync(tmp, s));
        return FM_OK;
    }
    return velocity_scan(G, E, t0, t1, j0, j1, d_out4, d_envelope, stream, false);
}

static int32_t velocity_scan(fm_grid G, fm_env E, int32_t t0, int32_t t1, int32_t j0, int32_t j1, double *d_out2,
                             int32_t *d_envelope, void *stream, bool exact)
{
    if (G.nx < 1 || G.ny < 1 || G.nt < 1 || E.n_real < 1 || E.n_modes < 0)
        return fm_fail(FM_BAD_ARG, "fm_velocity_max: bad dims");
    if (j0 < 0 || j1 > G.ny || j0 >= j1) return fm_fail(FM_BAD_ARG, "fm_velocity_max_rows: bad row range");
    if (t0 < 0 || t1 > G.nt || t0 >= t1) return fm_fail(FM_BAD_ARG, "fm_velocity_max_slab: bad layer range");
    cudaStream_t s = (cudaStream_t)stream;
    pool_keep();
    const int nc = (j1 - j0) * G.nx;   // cells scanned
    const int nm = E.n_modes;
    const int nts = t1 - t0;           // layers scanned
    int4 *vr = reinterpret_cast<int4 *>(d_envelope);
    if (nm > 16) {
        const int bxf = (nc + 255) / 256;
        const long long basef = (long long)bxf * nts, want = 4LL * sm_count();
        int rpb = E.n_real;
        if (basef < want) rpb = (int)((E.n_real + (want + basef - 1) / basef - 1) / ((want + basef - 1) / basef));
        if (rpb < 1) rpb = 1;
        const int nz = (E.n_real + rpb - 1) / rpb;
        if (vr && nz > 1) {
            k_envelope_init<<<(unsigned)(((long long)nts * nc + 255) / 256), 256, 0, s>>>(vr, G.nx * G.ny, t0, nts,
                                                                                          j0 * G.nx, nc);
            FM_CK_LAUNCH("k_envelope_init");
        }
        k_vmax_f64<8><<<dim3(bxf, nts, nz), 256, 0, s>>>(G, E, t0, j0 * G.nx, nc, rpb, d_out2, vr);
        FM_CK_LAUNCH("k_vmax_f64");
        return FM_OK;
    }
    // max_r |coeff[t, r, m]| per (t, m) of the slab: the error-bound ingredient
    double *cmax = nullptr;
    FM_CK(cudaMallocAsync(&cmax, sizeof(double) * (size_t)(nts * (nm > 0 ? nm : 1)), s));
    if (nm > 0) {
        k_maxabs_seg<<<nts * nm, 256, 0, s>>>(E.coeffs + (size_t)t0 * E.n_real * nm, E.n_real, nm, nm,
                                              (int64_t)E.n_real * nm, 1, cmax);
        FM_CK_LAUNCH("k_maxabs_seg");
    }
    if (!exact && nm <= 8 && getenv("FM_TC_SCAN")) {
        // bounds + envelope on the tensor cores (k_vmax_tc, opt-in): 64 cells
        // per block.  Measured at C2 (one B200): 4.23 ms vs 4.05 ms for the
        // FFMA2 scan -- the legacy mma.sync TF32 path issues ~1 m16n8k8 per
        // 21 cycles per SMSP, so the 3xTF32 split costs as much as the FFMA2
        // chains it replaces; the FFMA2 scan stays the default (its bound is
        // also 10x tighter)
        const int cpb = 8 * kTcQuads * 4;
        const int bxt = (nc + cpb - 1) / cpb;
        const long long baset = (long long)bxt * nts, wantt = 8LL * sm_count();
        int rpbt = E.n_real;
        if (baset < wantt) {
            const long long split = (wantt + baset - 1) / baset;
            rpbt = (int)((E.n_real + split - 1) / split);
            rpbt = ((rpbt + kTcChunk - 1) / kTcChunk) * kTcChunk;
        }
        const dim3 gridt(bxt, nts, (E.n_real + rpbt - 1) / rpbt);
        if (vr && gridt.z > 1) {
            k_envelope_init<<<(unsigned)(((long long)nts * nc + 255) / 256), 256, 0, s>>>(vr, G.nx * G.ny, t0, nts,
                                                                                          j0 * G.nx, nc);
            FM_CK_LAUNCH("k_envelope_init");
        }
        k_vmax_tc<<<gridt, 256, 0, s>>>(G, E, t0, j0 * G.nx, nc, rpbt, cmax, d_out2, vr);
        FM_CK_LAUNCH("k_vmax_tc");
        FM_CK(cudaFreeAsync(cmax, s));
        return FM_OK;
    }
    const int bx = (nc + 256 * kVmaxCells - 1) / (256 * kVmaxCells);
    long long base = (long long)bx * nts;
    int rpb = E.n_real;
    const long long want = 4LL * sm_count();
    if (base < want) {
        const long long split = (want + base - 1) / base;
        rpb = (int)((E.n_real + split - 1) / split);
        rpb = ((rpb + kVmaxChunk - 1) / kVmaxChunk) * kVmaxChunk;
    }
    dim3 grid(bx, nts, (E.n_real + rpb - 1) / rpb);
    if (vr && grid.z > 1) {
        k_envelope_init<<<(unsigned)(((long long)nts * nc + 255) / 256), 256, 0, s>>>(vr, G.nx * G.ny, t0, nts,
                                                                                      j0 * G.nx, nc);
        FM_CK_LAUNCH("k_envelope_init");
    }
    if (!exact) {
        if (nm <= 4)
            k_vmax<4, false><<<grid, 256, 0, s>>>(G, E, t0, j0 * G.nx, nc, rpb, cmax, d_out2, vr);
        else if (nm <= 8)
            k_vmax<8, false><<<grid, 256, 0, s>>>(G, E, t0, j0 * G.nx, nc, rpb, cmax, d_out2, vr);
        else
            k_vmax<16, false><<<grid, 256, 0, s>>>(G, E, t0, j0 * G.nx, nc, rpb, cmax, d_out2, vr);
    } else if (nm <= 4)
        k_vmax<4><<<grid, 256, 0, s>>>(G, E, t0, j0 * G.nx, nc, rpb, cmax, d_out2, vr);
    else if (nm <= 8)
        k_vmax<8><<<grid, 256, 0, s>>>(G, E, t0, j0 * G.nx, nc, rpb, cmax, d_out2, vr);
    else
        k_vmax<16><<<grid, 256, 0, s>>>(G, E, t0, j0 * G.nx, nc, rpb, cmax, d_out2, vr);
    FM_CK_LAUNCH("k_vmax");
    FM_CK(cudaFreeAsync(cmax, s));
    return FM_OK;
}

// ---------------------------------------------------------------------------
// segmented max-abs (velocity_bound ingredients, environment.py:404-419)
// ---------------------------------------------------------------------------
__global__ void k_maxabs_seg(const double *src, int64_t seg_len, int64_t elem_stride, int64_t inner,
                             int64_t outer_stride, int64_t inner_stride, double *out)
{
    const int64_t s = blockIdx.x;
    const double *b = src + (s / inner) * outer_stride + (s % inner) * inner_stride;
    double m = 0.0;
    for (int64_t k = threadIdx.x; k < seg_len; k += blockDim.x) m = nan_max(m, fabs(b[k * elem_stride]));
    m = warp_max_f64(m);
    __shared__ double red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        m = warp_max_f64(m);
        if (threadIdx.x == 0) out[s] = m;
    }
}

extern "C" int32_t fm_maxabs_segments(const double *src, int64_t n_seg, int64_t seg_len, int64_t elem_stride,
                                      int64_t inner, int64_t outer_stride, int64_t inner_stride,
                                      double *d_out, void *stream)
{
    if (n_seg <= 0) return FM_OK;
    if (inner < 1 || n_seg > 2147483647LL) return fm_fail(FM_BAD_ARG, "fm_maxabs_segments: bad shape");
    k_maxabs_seg<<<(unsigned)n_seg, 256, 0, (cudaStream_t)stream>>>(src, seg_len, elem_stride, inner,
                                                                      outer_stride, inner_stride, d_out);
    FM_CK_LAUNCH("k_maxabs_seg");
    return FM_OK;
}

// ---------------------------------------------------------------------------
// obstacle-mask summed-area tables: sat[t][(j+1)*(nx+1) + (i+1)]
// ---------------------------------------------------------------------------
__global__ void k_mask_sat(const uint8_t *mask, int nt, int ny, int nx, int32_t *sat)
{
    const int t = blockIdx.x;
    const uint8_t *m = mask + (size_t)t * nx * ny;
    int32_t *S = sat + (size_t)t * (nx + 1) * (ny + 1);
    const int W = nx + 1;
    for (int i = threadIdx.x; i <= nx; i += blockDim.x) S[i] = 0;
    for (int j = threadIdx.x; j < ny; j += blockDim.x) {
        int32_t run = 0;
        S[(j + 1) * W] = 0;
        for (int i = 0; i < nx; ++i) {
            run += m[j * nx + i] ? 1 : 0;
            S[(j + 1) * W + i + 1] = run;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
        int32_t run = 0;
        for (int j = 0; j < ny; ++j) {
            run += S[(j + 1) * W + i + 1];
            S[(j + 1) * W + i + 1] = run;
        }
    }
}

extern "C" int32_t fm_mask_sat(const uint8_t *mask, int32_t nt, int32_t ny, int32_t nx, int32_t *sat,
                               void *stream)
{
    if (nt < 1 || ny < 1 || nx < 1) return fm_fail(FM_BAD_ARG, "fm_mask_sat: bad dims");
    k_mask_sat<<<nt, 256, 0, (cudaStream_t)stream>>>(mask, nt, ny, nx, sat);
    FM_CK_LAUNCH("k_mask_sat");
    return FM_OK;
}

// ---------------------------------------------------------------------------
// K_build
// ---------------------------------------------------------------------------
// F_PROVEN: the host proved (fm_build_args.vmax_*) that every in-domain
//   landing lies inside the row's sub-grid window and every cell coordinate
//   fits in 2^30 -> lean rows need no window test and floor by magic add.
// F_CNT: the host proved every reward value dyadic with an exact sequential
//   sum -> lean rows form the reward sum from the histogram counts.
// F_GHIST: the sub-grid's per-warp histogram does not fit in shared memory
//   -> it lives in a global scratch slice per resident warp (same [slot][lane]
//   u16 layout, coalesced), fully checked rows only.
enum : int {
    F_DT_ONE = 1, F_OX_ZERO = 2, F_DX_MUL = 4, F_DX_ONE = 8, F_NET = 16, F_PROVEN = 32, F_CNT = 64, F_GHIST = 128
};
enum : int { RF_DEAD = 1, RF_TERMINAL = 2, RF_GATE = 4, RF_LANDWIN = 8, RF_SEGWIN = 16 };

// Per-(cell, realization) binning of lean tasks (F_PROVEN | F_CNT).
//
// With p = dx / dt and z = v / p, the landing of action a from cell column
// ci is ci + floor(z + c_a), c_a = 0.5 + a_x / p (model_builder.py:331-335
// in real arithmetic; x0 = origin + (ci + 0.5) dx, environment.py:99-100).
// Writing c_a = gamma_a + beta_a (integer + fraction), the displacement is
// gamma_a + floor(z) + [frac(z) >= theta_a], theta_a = 1 - beta_a: every
// action's landing is a step function of z whose steps sit at n + theta_a.
// The union of the theta_a (clustered, see bin_axis) cuts each unit of z
// into K + 1 sub-bins; a realization's bin (n, sub) in x and in y fixes its
// landing for EVERY action, so one 2-D histogram of bins per cell replaces
// the per-(cell, action, realization) work, and each row's counts are
// rectangle sums of it.  Exactness: z is computed in f32 with a rigorous
// error bound; a realization closer than the zone half-width to any step
// (or with any doubt) takes the exact f64 path of the reference instead
// (bin_drain), so the counts equal the reference's bit for bit.
static constexpr int kBinNS = 128;    // max buckets per unit interval of frac(z) (bin_ns: 32, 64 or 128)
static constexpr int kBinRep = 16;    // block-shared copies of each table entry (conflict-free lookups)
static constexpr int kBinMaxA = 64;   // actions with bin parameters
#ifndef FM_BIN_RING
#define FM_BIN_RING 4   // A/B at C2 with 16 warps/SM: 4 chunks 16.4 ms, 8 chunks (12 warps/SM) 17.4 ms
#endif
static constexpr int kBinRing = FM_BIN_RING;   // coefficient chunks in flight (32 realizations each)
#ifndef FM_BIN_WORDS2
#define FM_BIN_WORDS2 896    // u32 bin counters per warp for two cells (lean bin-only launch: 4 blocks / SM)
#endif
static constexpr int kBinQ = 128;     // deferred exact realizations per warp
// obstacle tasks (bin_task<.., OB = true>): a smaller ring beside (not under)
// the dense histogram, and a larger queue drained whenever it fills up
static constexpr int kBinRingO = 4;
static constexpr int kBinQO = 256;
struct BinEnt {
    // the zone intersecting the bucket: frac in [lo, hi] -> exact path; the
    // low 6 mantissa bits of lo hold kb + 1, kb = the sub-bin below the zone
    // (or of the whole bucket): lo is rounded down first, so the zone only widens
    float lo, hi;
};
struct BinAct {
    int gx, rx, gy, ry;   // gamma and cluster index (0 = always, K+1 = never) per axis
};

struct BuildK {
    // grid
    int nx, ny, nt, nc;
    double dx, dt, ox, oy, inv_dx, half_dx, inv_half_dx;
    // env
    const double *mean, *modes, *coeffs, *g;
    const uint8_t *mask;
    const int32_t *sat;
    int nm, nr;
    // actions / rewards
    const fm_action *act;
    int na, obj;
    double h_cr, r_term, r_out;
    int tcell;
    // sub-grid
    int hx, hy, width, nslot, hw;
    int rx, ry;
    int src_cell_exact;      // floor((x0(c) - o) / dx) == c for every cell centre
    // F_PROVEN: source columns / rows whose transit end ex = x0 + (x1 - x0)
    // equals x1 for every landing (Sterbenz): c >= lo or c <= hi
    int sx_lo, sx_hi, sy_lo, sy_hi;
    const int32_t *gate_r;   // device [rx, ry] (fm_gate_radius) or null
    // task decomposition
    int t0, t1, cell0, ncell;   // strip = cells [cell0, cell0 + ncell) of each layer
    int CW, RW, AG, nag, groups, RC;
    long long n_tasks;
    // per-warp shared-memory carve-up (bytes)
    int smem_warp, off_vbuf, off_coef, off_modes, off_danger;
    int off_queue;   // PART 2 (F_PROVEN | F_CNT): deferred exact-test queue [kQueue]
    int off_hg;      // PART 1 (F_PROVEN | F_NET): h_cr * g[t+1] per (cell, window slot)
    // outputs: rows of the model's cells [mcell0, mcell0 + mncell)
    int mcell0, mncell;
    int reserve_sms;    // SMs' worth of blocks left free for other streams
    uint64_t *row_ptr;
    uint16_t *row_nnz;
    double *reward;
    uint32_t *entries;
    unsigned long long capacity;
    unsigned long long *nnz_counter;
    uint32_t *viol;
    unsigned int *task_counter;
    unsigned int *task_list, *task_list_n;   // tasks the bin-only launches could not bin (PART 0 list launch)
    // PART 3 / 4: the tasks of the launch from k_classify's lists: list a,
    // then list b (PART 4: obstacle tasks near the obstacle first -- the
    // longest ones -- then the rest)
    const unsigned int *src_a, *src_b, *src_a_n, *src_b_n;
    uint16_t *ghist;   // F_GHIST: [resident warp][nslot + 1][32]
    // ---- per-(cell, realization) binning of lean tasks (see bin_task) ----
    int bin_ok;                 // the launch has bin tables (PART 1 lean tasks use them)
    int dev_flags;              // development A/B switches (FM_DEV_FLAGS; 0 in production)
    int bin_k1x, bin_k1y;       // sub-bins per unit of z = v / p, per axis (clusters + 1)
    int bin_p1;                 // p = dx / dt == 1 (z = v)
    float bin_ip;               // f32(1 / p)
    double bin_p;               // p
    double bin_dzone;           // zone half-width in z units (per-cell error must not exceed it)
    double bin_eps;             // allowance for the reference's own landing roundings (z units)
    int bin_words;              // u32 bin counters per warp
    int off_block;              // block-shared bytes before the warps' regions (bin tables)
    int off_bins, off_bdense, off_bq;   // per-warp regions of the bin path (union with the legacy ones):
                                        // counters | coefficient ring, later the dense histogram | queue
    int off_bring;                      // the coefficient ring (= off_bdense for lean tasks; separate for
                                        // obstacle tasks, which drain into the dense histogram mid-loop)
    const float *coef32;        // [t - t0][nr_pad][8] f32 coefficients (zero padded), per launch
    int nr_pad;                 // realizations rounded up to whole bin-loop iterations (64 by default)
    const double *cmax;         // [t - t0][nm] max_r |coeff[t, r, m]|
    const int4 *envelope;       // [nt][nc] per-cell velocity envelope (fm_velocity_scan) or null
    int bin_ns;                 // buckets per unit of frac(z): the smallest of 32 / 64 / 128 giving the same zones
    BinEnt tab[2 * (kBinNS + 1)];   // bucket tables, x then y, stride kBinNS + 1 (entry NS: frac == 1)
    BinAct bact[kBinMaxA];      // per action: (gamma_x, cluster r_x, gamma_y, r_y)
};

// fl(q / n) for 0 <= q <= n <= kFracMaxN at g_frac[n (n + 1) / 2 + q]: the
// segment-sampling fractions of environment.py:361 without a division each
static constexpr int kFracMaxN = 96;
__device__ double g_frac[(kFracMaxN + 1) * (kFracMaxN + 2) / 2];

static int32_t frac_table_init()
{
    static int dev_done = -1;
    int dev = 0;
    FM_CK(cudaGetDevice(&dev));
    if (dev_done == dev) return FM_OK;
    std::vector<double> h((kFracMaxN + 1) * (kFracMaxN + 2) / 2);
    for (int n = 1; n <= kFracMaxN; ++n)
        for (int q = 0; q <= n; ++q) h[n * (n + 1) / 2 + q] = (double)q / (double)n;   // IEEE, correctly rounded
    FM_CK(cudaMemcpyToSymbol(g_frac, h.data(), h.size() * sizeof(double)));
    dev_done = dev;
    return FM_OK;
}

// count of set mask cells at layer t inside [i0,i1] x [j0,j1] (clipped)
__device__ __forceinline__ int box_count(const BuildK &K, int t, int i0, int i1, int j0, int j1)
{
    i0 = max(i0, 0);
    j0 = max(j0, 0);
    i1 = min(i1, K.nx - 1);
    j1 = min(j1, K.ny - 1);
    if (i0 > i1 || j0 > j1) return 0;
    const int W = K.nx + 1;
    const int32_t *S = K.sat + (size_t)t * W * (K.ny + 1);
    return S[(j1 + 1) * W + i1 + 1] - S[j0 * W + i1 + 1] - S[(j1 + 1) * W + i0] + S[j0 * W + i0];
}

// floor(u) for |u| < 2^31 by one round-down add of 1.5 * 2^52 (the F2I
// conversion runs on the XU pipe at a quarter of the FP64 rate)
__device__ __forceinline__ int floor_magic(double u)
{
    return __double2loint(__dadd_rd(u, 6755399441055744.0));
}

// (x - origin) / dx with the reference's rounding (model_builder.py:333-334);
// the flags drop operations that are exact identities for this grid.
template <int FLAGS>
__device__ __forceinline__ double to_cell(double x, double o, double dx, double inv_dx)
{
    const double u = (FLAGS & F_OX_ZERO) ? x : DSUB(x, o);
    if (FLAGS & F_DX_ONE) return u;
    return (FLAGS & F_DX_MUL) ? DMUL(u, inv_dx) : DDIV(u, dx);
}

// _segments_blocked for one segment (environment.py:338-368), preceded by
// an exact-conservative bounding-box test against the mask SAT: samples are
// monotone in frac, so every sample cell lies in the box spanned by p0 and
// fl(p0 + delta); an empty box cannot block.
template <int FLAGS>
__device__ __forceinline__ bool seg_blocked(const BuildK &K, int t, double p0x, double p0y, double p1x, double p1y)
{
    const double ddx = DSUB(p1x, p0x), ddy = DSUB(p1y, p0y);
    const double ex = DADD(p0x, ddx), ey = DADD(p0y, ddy);
    const int ilo = __double2int_rd(to_cell<FLAGS>(fmin(p0x, ex), K.ox, K.dx, K.inv_dx));
    const int ihi = __double2int_rd(to_cell<FLAGS>(fmax(p0x, ex), K.ox, K.dx, K.inv_dx));
    const int jlo = __double2int_rd(to_cell<FLAGS>(fmin(p0y, ey), K.oy, K.dx, K.inv_dx));
    const int jhi = __double2int_rd(to_cell<FLAGS>(fmax(p0y, ey), K.oy, K.dx, K.inv_dx));
    if (box_count(K, t, ilo, ihi, jlo, jhi) == 0) return false;
    const double len = fm_hypot(ddx, ddy);
    double ns = ceil(DDIV(len, K.half_dx));
    if (!(ns >= 1.0)) ns = 1.0;
    const long long n = (long long)ns;
    FM_STAT(1, 1);
    FM_STAT(2, n + 1);
    const uint8_t *mt = K.mask + (size_t)t * K.nc;
    const double *ftab = n <= kFracMaxN ? g_frac + n * (n + 1) / 2 : nullptr;
    for (long long q = 0; q <= n; ++q) {
        // fl(q / n): tabulated correctly rounded quotients for small n
        double frac = ftab ? ftab[q] : DDIV((double)q, ns);
        if (frac > 1.0) frac = 1.0;
        const double px = DADD(p0x, DMUL(frac, ddx));
        const double py = DADD(p0y, DMUL(frac, ddy));
        const long long i = __double2ll_rd(to_cell<FLAGS>(px, K.ox, K.dx, K.inv_dx));
        const long long j = __double2ll_rd(to_cell<FLAGS>(py, K.oy, K.dx, K.inv_dx));
        if (i >= 0 && i < K.nx && j >= 0 && j < K.ny && mt[j * K.nx + i]) return true;
    }
    return false;
}

// The sampling part of _segments_blocked (environment.py:353-367) without
// the box prefilter, for segments already known to need it.
template <int FLAGS>
__device__ __forceinline__ bool seg_samples_blocked(const BuildK &K, int t, double p0x, double p0y, double p1x,
                                                    double p1y)
{
    const double ddx = DSUB(p1x, p0x), ddy = DSUB(p1y, p0y);
    if (FLAGS & F_PROVEN) {   // finite: the last sample first (see seg_samples_blocked_win)
        const int i = floor_magic(to_cell<FLAGS>(DADD(p0x, ddx), K.ox, K.dx, K.inv_dx));
        const int j = floor_magic(to_cell<FLAGS>(DADD(p0y, ddy), K.oy, K.dx, K.inv_dx));
        if ((unsigned)i < (unsigned)K.nx && (unsigned)j < (unsigned)K.ny &&
            __ldg(K.mask + (size_t)t * K.nc + j * K.nx + i))
            return true;
    }
    const double len = fm_hypot(ddx, ddy);
    double ns = ceil(DDIV(len, K.half_dx));
    if (!(ns >= 1.0)) ns = 1.0;
    const long long n = (long long)ns;
    FM_STAT(1, 1);
    FM_STAT(2, n + 1);
    const uint8_t *mt = K.mask + (size_t)t * K.nc;
    const double *ftab = n <= kFracMaxN ? g_frac + n * (n + 1) / 2 : nullptr;
    for (long long q = 0; q <= n; ++q) {
        double frac = ftab ? ftab[q] : DDIV((double)q, ns);
        if (frac > 1.0) frac = 1.0;
        const double px = DADD(p0x, DMUL(frac, ddx));
        const double py = DADD(p0y, DMUL(frac, ddy));
        const long long i = __double2ll_rd(to_cell<FLAGS>(px, K.ox, K.dx, K.inv_dx));
        const long long j = __double2ll_rd(to_cell<FLAGS>(py, K.oy, K.dx, K.inv_dx));
        if (i >= 0 && i < K.nx && j >= 0 && j < K.ny && __ldg(mt + j * K.nx + i)) return true;
    }
    return false;
}

// seg_samples_blocked for an obstacle bin task: the segment-sampling
// fractions fl(q / n) for n <= kFracSmemN from a block-shared copy of the
// table, and the mask at t from a per-cell shared window of cells
// [ci - hx - 1, ci + hx + 1] x [cj - hy - 1, cj + hy + 1] (every sample of a
// landing inside the sub-grid window lies in it: the samples are monotone
// between x0 and the transit end, which is within one cell of the landing);
// anything outside falls back to global memory.  Same arithmetic as
// environment.py:353-367.
static constexpr int kFracSmemN = 16;
template <int FLAGS>
__device__ __forceinline__ bool seg_samples_blocked_win(const BuildK &K, const double *ftab_s, const uint8_t *mwin,
                                                        int wi0, int wj0, int ww, int wh, int t, double p0x,
                                                        double p0y, double p1x, double p1y)
{
    const double ddx = DSUB(p1x, p0x), ddy = DSUB(p1y, p0y);
    {
        // the last sample first (frac = min(q / n, 1) = 1 exactly at q = n:
        // p0 + 1 * delta, environment.py:360-362): the test is an OR over the
        // samples, so an early exit on it is exact.  Most gated transitions
        // land on a cell the moving obstacle still covers at t -- they end
        // here without the hypot and the sample loop.
        const int i = floor_magic(to_cell<FLAGS>(DADD(p0x, ddx), K.ox, K.dx, K.inv_dx));
        const int j = floor_magic(to_cell<FLAGS>(DADD(p0y, ddy), K.oy, K.dx, K.inv_dx));
        if ((unsigned)i < (unsigned)K.nx && (unsigned)j < (unsigned)K.ny) {
            const int li = i - wi0, lj = j - wj0;
            if (((unsigned)li < (unsigned)ww && (unsigned)lj < (unsigned)wh)
                    ? mwin[lj * ww + li] != 0
                    : __ldg(K.mask + (size_t)t * K.nc + j * K.nx + i) != 0)
                return true;
        }
    }
    const double len = fm_hypot(ddx, ddy);
    // ceil(len / (0.5 dx)): for a power-of-two dx the quotient is an exact
    // scaling, so the product by the reciprocal rounds identically
    double ns = ceil((FLAGS & (F_DX_ONE | F_DX_MUL)) ? DMUL(len, K.inv_half_dx) : DDIV(len, K.half_dx));
    if (!(ns >= 1.0)) ns = 1.0;
    const long long n = (long long)ns;
    FM_STAT(1, 1);
    FM_STAT(2, n + 1);
    const uint8_t *mt = K.mask + (size_t)t * K.nc;
    const double *ftab = n <= kFracSmemN ? ftab_s + n * (n + 1) / 2 : n <= kFracMaxN ? g_frac + n * (n + 1) / 2 : nullptr;
    // four independent samples per step (early exit per step); coordinates
    // are below 2^30 cells (F_PROVEN), so floor is one round-down add
    for (long long q0 = 0; q0 <= n; q0 += 4) {
        bool hit = false;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long q = q0 + u;
            if (q <= n) {
                double frac = ftab ? ftab[q] : DDIV((double)q, ns);
                if (frac > 1.0) frac = 1.0;
                const double px = DADD(p0x, DMUL(frac, ddx));
                const double py = DADD(p0y, DMUL(frac, ddy));
                const int i = floor_magic(to_cell<FLAGS>(px, K.ox, K.dx, K.inv_dx));
                const int j = floor_magic(to_cell<FLAGS>(py, K.oy, K.dx, K.inv_dx));
                if ((unsigned)i < (unsigned)K.nx && (unsigned)j < (unsigned)K.ny) {
                    const int li = i - wi0, lj = j - wj0;
                    hit |= ((unsigned)li < (unsigned)ww && (unsigned)lj < (unsigned)wh)
                               ? mwin[lj * ww + li] != 0
                               : __ldg(mt + j * K.nx + i) != 0;
                }
            }
        }
        if (hit) return true;
    }
    return false;
}

struct SlowOut {
    double rw;
    int slot;
    int viol;
};

// Transitions the inline tiers cannot settle: an in-domain landing outside
// the sub-grid window (a sub-grid violation candidate) -- the full
// reference logic of step_flat + transition_sweep (model_builder.py:331-452).
// Reads its parameters from a global copy of BuildK so the call does not
// force the kernel-parameter block onto the stack.
template <int FLAGS>
__device__ __noinline__ SlowOut slow_step(const BuildK *__restrict__ Kg, int t, int ci, int cj, double x0, double y0,
                                          double x1, double y1, int i1, int j1, int rflags, double AB, double base,
                                          double base_hit)
{
    const BuildK &K = *Kg;
    const int di = i1 - ci, dj = j1 - cj;
    const bool inb = (unsigned)i1 < (unsigned)K.nx && (unsigned)j1 < (unsigned)K.ny;
    const bool inwin = (unsigned)(di + K.hx) <= (unsigned)(2 * K.hx) && (unsigned)(dj + K.hy) <= (unsigned)(2 * K.hy);
    const int succ = j1 * K.nx + i1;
    bool bad = !inb;
    if (inb) bad = K.mask[(size_t)(t + 1) * K.nc + succ] != 0;                      // landed in an obstacle
    if (!bad && (rflags & RF_GATE)) bad = seg_blocked<FLAGS>(K, t, x0, y0, x1, y1);  // transit
    SlowOut o;
    o.viol = (!bad && !inwin);
    const bool hit = !bad && succ == K.tcell;
    if (K.obj == FM_OBJ_NET_ENERGY) {
        const double gd = inb ? K.g[(size_t)(t + 1) * K.nc + succ] : 0.0;
        const double b = DMUL(DADD(AB, DMUL(K.h_cr, gd)), K.dt);
        o.rw = hit ? DADD(b, K.r_term) : b;
    } else {
        o.rw = hit ? base_hit : base;
    }
    o.slot = (bad || !inwin) ? K.nslot : (dj + K.hy) * K.width + (di + K.hx);
    if (bad) o.rw = K.r_out;
    return o;
}

template <int FLAGS>
__device__ __noinline__ bool seg_blocked_call(const BuildK *__restrict__ Kg, int t, double p0x, double p0y, double p1x,
                                              double p1y)
{
    return seg_blocked<FLAGS>(*Kg, t, p0x, p0y, p1x, p1y);
}

__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gmem_src)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Per-row constants of one task (registers).
struct RowC {
    double x0, y0, ax, ay, base, base_hit, AB;
    int ci, cj, ilc, jlc, wi, wj, soff, tslot, rflags;
};

// One transition of one row (step_flat + the slot / dead logic of
// transition_sweep).  OBST = some row of this warp is dead or has an
// obstacle cell near it; otherwise none of the obstacle tests can fire and
// the lean variant is exact.
//   tier 1: landing inside the row's grid-clipped sub-grid window
//   tier 2: landing outside the domain -> SINK, r_outbound
//   tier 3: in-domain landing outside the window -> slow_step
template <int FLAGS, bool OBST>
__device__ __forceinline__ void step_one(const BuildK &K, const BuildK *__restrict__ Kg, int t, const RowC &R,
                                         const double2 v, const double *__restrict__ g_n,
                                         const uint8_t *__restrict__ mask_n, int &slot, double &rw, int &viol)
{
    double px = DADD(v.x, R.ax), py = DADD(v.y, R.ay);   // x' = x0 + (v + a) * dt  (model_builder.py:332)
    if (!(FLAGS & F_DT_ONE)) {
        px = DMUL(px, K.dt);
        py = DMUL(py, K.dt);
    }
    const double x1 = DADD(R.x0, px), y1 = DADD(R.y0, py);
    const int i1 = __double2int_rd(to_cell<FLAGS>(x1, K.ox, K.dx, K.inv_dx));
    const int j1 = __double2int_rd(to_cell<FLAGS>(y1, K.oy, K.dx, K.inv_dx));
    if ((unsigned)(i1 - R.ilc) <= (unsigned)R.wi && (unsigned)(j1 - R.jlc) <= (unsigned)R.wj) {
        slot = j1 * K.width + i1 + R.soff;
        bool bad = false;
        if (OBST) {
            if (R.rflags & RF_LANDWIN) bad = mask_n[j1 * K.nx + i1] != 0;
            if (!bad && (R.rflags & RF_SEGWIN)) {
                // every sample cell of the segment lies within one cell of the
                // box spanned by the source and landing cells
                if (box_count(K, t, min(R.ci, i1) - 1, max(R.ci, i1) + 1, min(R.cj, j1) - 1, max(R.cj, j1) + 1) > 0)
                    bad = seg_blocked_call<FLAGS>(Kg, t, R.x0, R.y0, x1, y1);
            }
        }
        const bool hit = !bad && slot == R.tslot;
        if (FLAGS & F_NET) {
            const double gd = __ldg(g_n + j1 * K.nx + i1);
            double b = DADD(R.AB, DMUL(K.h_cr, gd));
            if (!(FLAGS & F_DT_ONE)) b = DMUL(b, K.dt);
            rw = hit ? DADD(b, K.r_term) : b;
        } else {
            rw = hit ? R.base_hit : R.base;
        }
        if (OBST && bad) {
            slot = K.nslot;
            rw = K.r_out;
        }
    } else if ((unsigned)i1 >= (unsigned)K.nx || (unsigned)j1 >= (unsigned)K.ny) {
        slot = K.nslot;   // left the domain
        rw = K.r_out;
    } else {
        const SlowOut o = slow_step<FLAGS>(Kg, t, R.ci, R.cj, R.x0, R.y0, x1, y1, i1, j1, R.rflags, R.AB, R.base,
                                           R.base_hit);
        slot = o.slot;
        rw = o.rw;
        viol |= o.viol;
    }
    if (OBST && (R.rflags & RF_DEAD)) {   // after the overflow check (model_builder.py:445-452)
        slot = K.nslot;
        rw = (R.rflags & RF_TERMINAL) ? 0.0 : K.r_out;
    }
}

// u16 counters laid out [slot][lane]: one IMAD + LDS.U16 + IADD + STS.U16
// The full per-transition logic (tiers of step_one with obstacle handling)
// for the rare transitions the branch-free fast path cannot settle.
// Returns the slot relative to the row's window origin (q = slot - soff).
template <int FLAGS>
__device__ __noinline__ SlowOut rare_transition(const BuildK *__restrict__ Kg, int t, const RowC R, const double2 v)
{
    const BuildK &K = *Kg;
    FM_STAT(0, 1);
    const double *g_n = K.g + (size_t)(t + 1) * K.nc;
    const uint8_t *mask_n = K.mask + (size_t)(t + 1) * K.nc;
    SlowOut o;
    o.viol = 0;
    RowC Ra = R;   // fast-path form -> absolute target slot
    Ra.tslot = R.tslot == INT_MIN ? -1 : R.tslot + R.soff;
    step_one<FLAGS, true>(K, Kg, t, Ra, v, g_n, mask_n, o.slot, o.rw, o.viol);
    o.slot -= R.soff;
    return o;
}

// floor(u) for |u| < 2^31: u + 1.5*2^52 lies in [2^52, 2^53) where the ulp
// is 1, so the round-down add is exactly 1.5*2^52 + floor(u); its low word
// is floor(u) in two's complement.  One DADD instead of an F2I (XU pipe,
// a quarter of the FP64 rate).

// Branch-free fast transition.  Valid when the landing is inside the row's
// grid-clipped window and (OBST) not on a danger slot of the row's cell --
// a cell masked at t+1 or a gated segment whose box touches the mask at t --
// or (EDGE) outside the domain (-> SINK).  Dead source rows (OBST) are
// overridden here; everything else goes to rare_transition.
template <int FLAGS, bool EDGE, bool OBST>
__device__ __forceinline__ bool fast_transition(const BuildK &K, const RowC &R, const double2 v,
                                                const double *__restrict__ g_n, const uint32_t *cls, int outq,
                                                int &q, double &rw)
{
    double px = DADD(v.x, R.ax), py = DADD(v.y, R.ay);   // x' = x0 + (v + a) * dt  (model_builder.py:332)
    if (!(FLAGS & F_DT_ONE)) {
        px = DMUL(px, K.dt);
        py = DMUL(py, K.dt);
    }
    const double x1 = DADD(R.x0, px), y1 = DADD(R.y0, py);
    int i1, j1;
    bool inwin;
    if (FLAGS & F_PROVEN) {
        // proven: an in-domain landing is inside the (clipped) window
        i1 = floor_magic(to_cell<FLAGS>(x1, K.ox, K.dx, K.inv_dx));
        j1 = floor_magic(to_cell<FLAGS>(y1, K.oy, K.dx, K.inv_dx));
        inwin = !EDGE || ((unsigned)i1 < (unsigned)K.nx && (unsigned)j1 < (unsigned)K.ny);
    } else {
        i1 = __double2int_rd(to_cell<FLAGS>(x1, K.ox, K.dx, K.inv_dx));
        j1 = __double2int_rd(to_cell<FLAGS>(y1, K.oy, K.dx, K.inv_dx));
        inwin = (unsigned)(i1 - R.ilc) <= (unsigned)R.wi && (unsigned)(j1 - R.jlc) <= (unsigned)R.wj;
    }
    q = j1 * K.width + i1;                       // slot - soff
    const bool hit = q == R.tslot;               // R.tslot holds tslot - soff
    if (FLAGS & F_NET) {
        const double gd = inwin ? __ldg(g_n + j1 * K.nx + i1) : 0.0;
        double b = DADD(R.AB, DMUL(K.h_cr, gd));
        if (!(FLAGS & F_DT_ONE)) b = DMUL(b, K.dt);
        rw = hit ? DADD(b, K.r_term) : b;
    } else {
        rw = hit ? R.base_hit : R.base;
    }
    bool ok = inwin;
    if (OBST) {
        const int slot = q + R.soff;
        // slot class (2 bits per slot, see the danger map in k_build):
        // 1 landing cell masked at t+1 -> bad whatever the transit
        //   (model_builder.py:336, 347), settled here;
        // 2 gated segment whose tight box (source cell x landing cell)
        //   touches the mask at t -> exact test;
        // 3 only the box grown by one cell touches it -> exact test only if
        //   the transit end ex = x0 + (x1 - x0) leaves the landing cell
        const int c = inwin ? (int)((cls[slot >> 4] >> ((slot & 15) << 1)) & 3u) : 0;
        const bool land = c == 1;
        bool segd = c == 2;
        if (c == 3) {
            const double ex = DADD(R.x0, DSUB(x1, R.x0)), ey = DADD(R.y0, DSUB(y1, R.y0));
            const int ei = __double2int_rd(to_cell<FLAGS>(ex, K.ox, K.dx, K.inv_dx));
            const int ej = __double2int_rd(to_cell<FLAGS>(ey, K.oy, K.dx, K.inv_dx));
            segd = ei != i1 || ej != j1;
        }
        const bool dead = R.rflags & RF_DEAD;
        ok = inwin && (!segd || dead);
        if (land) {
            q = outq;
            rw = K.r_out;
        }
        if (dead) {   // after the overflow check (model_builder.py:445-452)
            q = outq;
            rw = (R.rflags & RF_TERMINAL) ? 0.0 : K.r_out;
        }
    }
    if (EDGE) {
        const bool out = (unsigned)i1 >= (unsigned)K.nx || (unsigned)j1 >= (unsigned)K.ny;
        if (!inwin) {
            q = outq;
            rw = (OBST && (R.rflags & RF_TERMINAL)) ? 0.0 : K.r_out;
        }
        ok = ok || out;
    }
    return ok;
}

// Reconstruction of this recon lane's realizations of one chunk for 8 modes
// (environment.py:293-297: v = mean; v += c_m * mode_m for ascending m, two
// roundings per term): the cell's modes stay in registers, two
// realizations per pass share them, coefficients come as [pair][r] double2.
__device__ __forceinline__ void recon_m8(const double2 *md, const double2 *c2, double2 mu, int RC, int RW, int RPL,
                                         int rr, int n_left, double2 *vout)
{
    double2 m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = md[i];
    for (int p = 0; p < RPL; p += 2) {
        // odd RPL recomputes rl0; realizations past the chunk (RW not dividing
        // RC) read a valid coefficient and are not stored
        const int rl0 = p * RW + rr < RC ? p * RW + rr : RC - 1;
        const int rl1 = p + 1 < RPL && rl0 + RW < RC ? rl0 + RW : rl0;
        double x0 = mu.x, y0 = mu.y, x1 = mu.x, y1 = mu.y;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 k0 = c2[q * RC + rl0], k1 = c2[q * RC + rl1];
            x0 = DADD(x0, DMUL(k0.x, m[2 * q].x));
            y0 = DADD(y0, DMUL(k0.x, m[2 * q].y));
            x1 = DADD(x1, DMUL(k1.x, m[2 * q].x));
            y1 = DADD(y1, DMUL(k1.x, m[2 * q].y));
            x0 = DADD(x0, DMUL(k0.y, m[2 * q + 1].x));
            y0 = DADD(y0, DMUL(k0.y, m[2 * q + 1].y));
            x1 = DADD(x1, DMUL(k1.y, m[2 * q + 1].x));
            y1 = DADD(y1, DMUL(k1.y, m[2 * q + 1].y));
        }
        if (p * RW + rr < RC && rl0 < n_left) vout[rl0] = make_double2(x0, y0);
        if (rl1 != rl0 && rl1 < n_left) vout[rl1] = make_double2(x1, y1);
    }
}

// One lean transition: landing slot q (OUT for a landing outside the domain
// in EDGE warps) and, unless F_CNT, its reward.
template <int FLAGS, bool EDGE>
__device__ __forceinline__ int lean_transition(const BuildK &K, const RowC &R, const double2 v,
                                               const double *__restrict__ g_n, int outq, double &rw)
{
    double px = DADD(v.x, R.ax), py = DADD(v.y, R.ay);   // x' = x0 + (v + a) * dt  (model_builder.py:332)
    if (!(FLAGS & F_DT_ONE)) {
        px = DMUL(px, K.dt);
        py = DMUL(py, K.dt);
    }
    const int i1 = floor_magic(to_cell<FLAGS>(DADD(R.x0, px), K.ox, K.dx, K.inv_dx));
    const int j1 = floor_magic(to_cell<FLAGS>(DADD(R.y0, py), K.oy, K.dx, K.inv_dx));
    int q = j1 * K.width + i1;
    // net energy: g_n here is the warp's table h_cr * g[t+1][landing cell]
    // per window slot, shifted by soff (0 for cells outside the domain); read
    // at the window slot, which exists for every landing under F_PROVEN
    const double hg = (FLAGS & F_NET) ? g_n[q] : 0.0;
    bool out = false;
    if (EDGE) {
        out = (unsigned)i1 >= (unsigned)K.nx || (unsigned)j1 >= (unsigned)K.ny;
        if (out) q = outq;
    }
    if (!(FLAGS & F_CNT)) {
        const bool hit = q == R.tslot;
        if (FLAGS & F_NET) {
            double b = DADD(R.AB, hg);
            if (!(FLAGS & F_DT_ONE)) b = DMUL(b, K.dt);
            rw = hit ? DADD(b, K.r_term) : b;
        } else {
            rw = hit ? R.base_hit : R.base;
        }
        if (EDGE && out) rw = K.r_out;
    }
    return q;
}

// Shared-memory reductions for the lean histogram updates are the default
// (A/B at C2: 103 ms vs 111 ms for load/add/store, whose dependency chain
// serialises the 8 updates of a batch); -DFM_HIST_RMW selects the latter.
#if !defined(FM_HIST_RMW) && !defined(FM_HIST_ATOMS)
#define FM_HIST_ATOMS
#endif

// Histogram increment of this lane's u16 counter [q][lane].  FM_HIST_ATOMS:
// a 32-bit shared-memory reduction on the word holding the counter
// (hs_word = shared address of that word for q = 0; no read-modify-write
// dependency chain; counts <= n_real <= 65535 never carry into the
// neighbouring lane's half).
__device__ __forceinline__ void hist_inc(uint16_t *h16q, unsigned hs_word, int q, unsigned half_one)
{
#ifdef FM_HIST_ATOMS
    (void)h16q;
    // no memory clobber: the velocity loads of the next batch may be hoisted
    // above these reductions (they never alias the histogram); the callers
    // fence the compiler before the histogram is read with plain loads
    asm volatile("red.shared.add.u32 [%0], %1;\n" ::"r"(hs_word + (unsigned)q * 64u), "r"(half_one));
#else
    (void)hs_word;
    h16q[q * 32] += (uint16_t)((half_one & 0xFFFFu) | (half_one >> 16));   // the increment, whichever half
#endif
}

// The realization loop of one chunk for lean rows under F_PROVEN: no
// obstacle near the warp's rows, every landing inside the window or (EDGE
// warps) outside the domain -> SINK.  No vote, no rare path.  Reward sum in
// ascending realization order unless F_CNT (then formed from the counts).
// Velocities of U realizations are loaded before any histogram store so the
// shared loads are not ordered behind possibly-aliasing stores.
template <int FLAGS, bool EDGE>
__device__ __forceinline__ void chunk_rows_lean(const BuildK &K, const RowC &R, const double2 *vrow, int nk,
                                                const double *__restrict__ g_n, uint16_t *h16q, int outq, double &S,
                                                unsigned half_one)
{
    const unsigned hs_word = (unsigned)__cvta_generic_to_shared(h16q) & ~3u;
#ifndef FM_LEAN_U
#define FM_LEAN_U 8
#endif
    constexpr int U = FM_LEAN_U;
    int k = 0;
#ifndef FM_LEAN_NO_FULL
    // (count-formed rewards only: with a per-transition reward chain the
    // unrolled chunk spills)
    if ((FLAGS & F_CNT) && nk == FM_BUILD_RC) {
        // full chunk: the batch loop unrolled (no loop-carried branch; the
        // scheduler may interleave consecutive batches)
#ifndef FM_LEAN_NO_PREFETCH
        // velocities of the next batch loaded before this batch's math
        double2 vn[U];
#pragma unroll
        for (int u = 0; u < U; ++u) vn[u] = vrow[u];
#endif
#pragma unroll
        for (int kb = 0; kb < FM_BUILD_RC; kb += U) {
            double2 v[U];
#ifndef FM_LEAN_NO_PREFETCH
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = vn[u];
            if (kb + U < FM_BUILD_RC) {
#pragma unroll
                for (int u = 0; u < U; ++u) vn[u] = vrow[kb + U + u];
            }
#else
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = vrow[kb + u];
#endif
            int q[U];
            double w[U];
#pragma unroll
            for (int u = 0; u < U; ++u) q[u] = lean_transition<FLAGS, EDGE>(K, R, v[u], g_n, outq, w[u]);
            if (!(FLAGS & F_CNT)) {
#pragma unroll
                for (int u = 0; u < U; ++u) S = DADD(S, w[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) hist_inc(h16q, hs_word, q[u], half_one);
        }
        return;
    }
#endif
    for (; k + U <= nk; k += U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = vrow[k + u];
        int q[U];
        double w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) q[u] = lean_transition<FLAGS, EDGE>(K, R, v[u], g_n, outq, w[u]);
        if (!(FLAGS & F_CNT)) {   // ascending realization order (model_builder.py:457-458)
#pragma unroll
            for (int u = 0; u < U; ++u) S = DADD(S, w[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) hist_inc(h16q, hs_word, q[u], half_one);
    }
    for (; k < nk; ++k) {
        double w0;
        const int q0 = lean_transition<FLAGS, EDGE>(K, R, vrow[k], g_n, outq, w0);
        if (!(FLAGS & F_CNT)) S = DADD(S, w0);
        hist_inc(h16q, hs_word, q0, half_one);
    }
}

// Landing slot of one transition in an obstacle warp under F_PROVEN | F_CNT
// (rewards come from the counts, so only the slot is needed).  Landings
// outside the domain stay in their (unclipped) window slot -- class 0 --
// and are folded into OUT in the epilogue; `rare` = exact segment test.
template <int FLAGS>
__device__ __forceinline__ int obst_slot(const BuildK &K, const RowC &R, const double2 v, const uint32_t *cls,
                                         int outq, bool &rare)
{
    double px = DADD(v.x, R.ax), py = DADD(v.y, R.ay);   // x' = x0 + (v + a) * dt  (model_builder.py:332)
    if (!(FLAGS & F_DT_ONE)) {
        px = DMUL(px, K.dt);
        py = DMUL(py, K.dt);
    }
    const double x1 = DADD(R.x0, px), y1 = DADD(R.y0, py);
    const int i1 = floor_magic(to_cell<FLAGS>(x1, K.ox, K.dx, K.inv_dx));
    const int j1 = floor_magic(to_cell<FLAGS>(y1, K.oy, K.dx, K.inv_dx));
    const int q = j1 * K.width + i1, slot = q + R.soff;
    const int c = (int)((cls[slot >> 4] >> ((slot & 15) << 1)) & 3u);   // see fast_transition
    // classes 2 and 3 are deferred to the exact sampling (for class 3 the
    // box prefilter would mostly clear it, but the few class-3 slots left
    // after the Sterbenz downgrade are not worth a branch per transition)
    rare = c >= 2;
    return c == 1 ? outq : q;
}

// A deferred exact segment test: transit end, owner lane, landing slot.
struct QItem {
    double x1, y1;
    int32_t meta;   // owner lane << 16 | landing slot (window index, < 65535)
};
static constexpr int kQueue = 64;

// Obstacle-warp realization loop under F_PROVEN | F_CNT for the live (not
// dead) rows.  Counts commute (rewards come from the counts), so exact
// segment tests are deferred to the end of the chunk and run by all lanes
// that have one at once -- one pass per pending item of the busiest lane --
// instead of one divergent call per batch position (the deferred items are
// marked in a 64-bit mask of chunk-local realizations).
template <int FLAGS>
__device__ __forceinline__ void chunk_rows_obst_cnt(const BuildK *__restrict__ Kg, int t, const RowC &R,
                                                    const double2 *vrow, int nk, const uint32_t *cls,
                                                    uint16_t *h16q, int outq, bool live, unsigned half_one,
                                                    unsigned char *qbase, unsigned hist_s, int grp)
{
    const BuildK &K = *Kg;
    const unsigned hs_word = (unsigned)__cvta_generic_to_shared(h16q) & ~3u;
    unsigned long long pend = 0;
    int k = live ? 0 : nk;
    for (; k + 4 <= nk; k += 4) {
        double2 v[4];
        int q[4];
        bool r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = vrow[k + u];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = obst_slot<FLAGS>(K, R, v[u], cls, outq, r[u]);
        // branch-free: a deferred transition adds 0 now (its slot is settled
        // in the drain); the batch's deferral bits enter the mask at once
#pragma unroll
        for (int u = 0; u < 4; ++u) hist_inc(h16q, hs_word, q[u], r[u] ? 0u : half_one);
        const unsigned bits = (r[0] ? 1u : 0u) | (r[1] ? 2u : 0u) | (r[2] ? 4u : 0u) | (r[3] ? 8u : 0u);
        pend |= (unsigned long long)bits << (k & 63);
    }
    for (; k < nk; ++k) {
        bool r0;
        const int q0 = obst_slot<FLAGS>(K, R, vrow[k], cls, outq, r0);
        if (r0) pend |= 1ull << (k & 63);
        else hist_inc(h16q, hs_word, q0, half_one);
    }
    // drain: the live lanes park their deferred transitions in the warp's
    // queue, then every lane of the warp takes queue entries round-robin
    // (the exact tests of one busy row are spread over all 32 lanes)
    QItem *queue = reinterpret_cast<QItem *>(qbase);
    const int lane = threadIdx.x & 31;
    for (;;) {
        const int mine = __popcll(pend);
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(kFull, incl, 31);
        if (total == 0) break;
        int pos = incl - mine;
        while (pend && pos < kQueue) {
            const int kk = __ffsll((long long)pend) - 1;
            pend &= pend - 1;
            const double2 v = vrow[kk];
            double px = DADD(v.x, R.ax), py = DADD(v.y, R.ay);
            if (!(FLAGS & F_DT_ONE)) {
                px = DMUL(px, K.dt);
                py = DMUL(py, K.dt);
            }
            const double x1 = DADD(R.x0, px), y1 = DADD(R.y0, py);
            const int q = floor_magic(to_cell<FLAGS>(y1, K.oy, K.dx, K.inv_dx)) * K.width +
                          floor_magic(to_cell<FLAGS>(x1, K.ox, K.dx, K.inv_dx));
            queue[pos].x1 = x1;
            queue[pos].y1 = y1;
            queue[pos].meta = (lane << 16) | (q + R.soff);
            ++pos;
        }
        __syncwarp();
        const int n_q = total < kQueue ? total : kQueue;
        for (int e = lane; e < n_q; e += 32) {
            // the deferred transition lands in-domain on an unmasked cell
            // (class 2/3): only the transit samples decide (env.py:353-367)
            const QItem it = queue[e];
            const int owner = it.meta >> 16, slot = it.meta & 0xFFFF;
            const int c = K.cell0 + grp * K.CW + owner / K.AG;
            const double x0 = DADD(K.ox, DMUL(DADD((double)(c % K.nx), 0.5), K.dx));   // environment.py:99-100
            const double y0 = DADD(K.oy, DMUL(DADD((double)(c / K.nx), 0.5), K.dx));
            const int sl = seg_samples_blocked<FLAGS>(K, t, x0, y0, it.x1, it.y1) ? K.nslot : slot;
            // the owner's u16 counter [slot][owner] lives in word (slot * 16 + owner / 2)
            asm volatile("red.shared.add.u32 [%0], %1;\n" ::"r"(hist_s + (unsigned)sl * 64u + (unsigned)(owner >> 1) * 4u),
                         "r"(1u << ((owner & 1) * 16))
                         : "memory");
        }
        __syncwarp();
    }
}

// Obstacle-warp realization loop under F_PROVEN without F_CNT (net_energy,
// or time / energy with non-dyadic rewards): the reward sum must follow the
// reference's realization order, so exact segment tests run in place.
// Branch-free slot classes; landings outside the domain, on a cell masked at
// t+1 or through a blocked transit are bad (SINK, r_outbound); dead rows
// send every realization to SINK (no overflow test is needed under
// F_PROVEN).  model_builder.py:331-360, 445-458; environment.py:338-368.
template <int FLAGS>
__device__ __forceinline__ void chunk_rows_obst_seq(const BuildK *__restrict__ Kg, int t, const RowC &R,
                                                    const double2 *vrow, int nk, const double *__restrict__ g_n,
                                                    const uint32_t *cls, uint16_t *h16q, int outq, unsigned rowmask,
                                                    double &S, unsigned half_one)
{
    const BuildK &K = *Kg;
    const unsigned hs_word = (unsigned)__cvta_generic_to_shared(h16q) & ~3u;
    const unsigned live = __ballot_sync(rowmask, !(R.rflags & RF_DEAD));
    if (R.rflags & RF_DEAD) {
        const double rw = (R.rflags & RF_TERMINAL) ? 0.0 : K.r_out;
        for (int k = 0; k < nk; ++k) S = DADD(S, rw);   // ascending realization order
        if (nk > 0) hist_inc(h16q, hs_word, outq, half_one * (unsigned)nk);
        return;
    }
    int k = 0;
    for (; k < nk; k += 4) {
        const int nb = nk - k < 4 ? nk - k : 4;
        double x1[4], y1[4];
        int q[4], cell[4];
        bool bad[4], rare[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double2 v = vrow[k + (u < nb ? u : 0)];
            double px = DADD(v.x, R.ax), py = DADD(v.y, R.ay);   // x' = x0 + (v + a) * dt  (model_builder.py:332)
            if (!(FLAGS & F_DT_ONE)) {
                px = DMUL(px, K.dt);
                py = DMUL(py, K.dt);
            }
            x1[u] = DADD(R.x0, px);
            y1[u] = DADD(R.y0, py);
            const int i1 = floor_magic(to_cell<FLAGS>(x1[u], K.ox, K.dx, K.inv_dx));
            const int j1 = floor_magic(to_cell<FLAGS>(y1[u], K.oy, K.dx, K.inv_dx));
            q[u] = j1 * K.width + i1;
            cell[u] = j1 * K.nx + i1;
            const bool out = (unsigned)i1 >= (unsigned)K.nx || (unsigned)j1 >= (unsigned)K.ny;
            const int slot = q[u] + R.soff;   // inside the window (F_PROVEN)
            const int c = out ? 0 : (int)((cls[slot >> 4] >> ((slot & 15) << 1)) & 3u);
            bad[u] = out || c == 1;
            rare[u] = u < nb && c >= 2;
        }
        if (!__all_sync(live, !(rare[0] || rare[1] || rare[2] || rare[3]))) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (rare[u]) bad[u] = seg_samples_blocked<FLAGS>(K, t, R.x0, R.y0, x1[u], y1[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (u >= nb) break;
            const bool hit = !bad[u] && q[u] == R.tslot;
            double rw;
            if (FLAGS & F_NET) {
                const double gd = bad[u] ? 0.0 : __ldg(g_n + cell[u]);
                double b = DADD(R.AB, DMUL(K.h_cr, gd));
                if (!(FLAGS & F_DT_ONE)) b = DMUL(b, K.dt);
                rw = hit ? DADD(b, K.r_term) : b;
            } else {
                rw = hit ? R.base_hit : R.base;
            }
            if (bad[u]) rw = K.r_out;
            S = DADD(S, rw);   // ascending realization order (model_builder.py:457-458)
            hist_inc(h16q, hs_word, bad[u] ? outq : q[u], half_one);
        }
    }
}

// The realization loop of one chunk for the row lanes: 4 independent
// transitions per iteration in straight-line code (interleaved by the
// compiler), one warp vote to divert rare lanes, reward sums in ascending r.
// h16q points at the row's histogram origin shifted by soff (q indexing).
template <int FLAGS, bool EDGE, bool OBST>
__device__ __forceinline__ void chunk_rows(const BuildK &K, const BuildK *__restrict__ Kg, int t, const RowC &R,
                                           const double2 *vrow, int nk, const double *__restrict__ g_n,
                                           const uint32_t *cls, uint16_t *h16q, int outq,
                                           unsigned rowmask, double &S, int &viol)
{
    int k = 0;
    for (; k + 4 <= nk; k += 4) {
        const double2 v0 = vrow[k], v1 = vrow[k + 1], v2 = vrow[k + 2], v3 = vrow[k + 3];
        int q0, q1, q2, q3;
        double w0, w1, w2, w3;
        const bool f0 = fast_transition<FLAGS, EDGE, OBST>(K, R, v0, g_n, cls, outq, q0, w0);
        const bool f1 = fast_transition<FLAGS, EDGE, OBST>(K, R, v1, g_n, cls, outq, q1, w1);
        const bool f2 = fast_transition<FLAGS, EDGE, OBST>(K, R, v2, g_n, cls, outq, q2, w2);
        const bool f3 = fast_transition<FLAGS, EDGE, OBST>(K, R, v3, g_n, cls, outq, q3, w3);
        if (!__all_sync(rowmask, f0 && f1 && f2 && f3)) {
            if (!f0) { const SlowOut o = rare_transition<FLAGS>(Kg, t, R, v0); q0 = o.slot; w0 = o.rw; viol |= o.viol; }
            if (!f1) { const SlowOut o = rare_transition<FLAGS>(Kg, t, R, v1); q1 = o.slot; w1 = o.rw; viol |= o.viol; }
            if (!f2) { const SlowOut o = rare_transition<FLAGS>(Kg, t, R, v2); q2 = o.slot; w2 = o.rw; viol |= o.viol; }
            if (!f3) { const SlowOut o = rare_transition<FLAGS>(Kg, t, R, v3); q3 = o.slot; w3 = o.rw; viol |= o.viol; }
        }
        S = DADD(S, w0);   // ascending realization order (model_builder.py:457-458)
        S = DADD(S, w1);
        S = DADD(S, w2);
        S = DADD(S, w3);
        h16q[q0 * 32] += (uint16_t)1;   // u16 counters [slot][lane]
        h16q[q1 * 32] += (uint16_t)1;
        h16q[q2 * 32] += (uint16_t)1;
        h16q[q3 * 32] += (uint16_t)1;
    }
    for (; k < nk; ++k) {
        int q0;
        double w0;
        const bool f0 = fast_transition<FLAGS, EDGE, OBST>(K, R, vrow[k], g_n, cls, outq, q0, w0);
        if (!f0) {
            const SlowOut o = rare_transition<FLAGS>(Kg, t, R, vrow[k]);
            q0 = o.slot;
            w0 = o.rw;
            viol |= o.viol;
        }
        S = DADD(S, w0);
        h16q[q0 * 32] += (uint16_t)1;
    }
}

// ---- per-(cell, realization) binning (lean tasks, F_PROVEN | F_CNT) --------

__device__ __forceinline__ unsigned long long f2_bits(float2 a) { return *reinterpret_cast<unsigned long long *>(&a); }
__device__ __forceinline__ float2 f2_from(unsigned long long r) { return *reinterpret_cast<float2 *>(&r); }
__device__ __forceinline__ float2 f2_add_rm(float2 a, float2 b)
{
    unsigned long long r;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_from(r);
}
__device__ __forceinline__ float2 f2_add(float2 a, float2 b)
{
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_from(r);
}
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b)
{
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_from(r);
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b)
{
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_from(r);
}
__device__ __forceinline__ float2 f2_fma_rm(float2 a, float2 b, float2 c)
{
    unsigned long long r;
    asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
    return f2_from(r);
}
__device__ __forceinline__ void cp_async_wait_ring() { asm volatile("cp.async.wait_group %0;\n" ::"n"(kBinRing - 1) : "memory"); }

// One cell of a bin task: f32 reconstruction inputs and the bin box.
struct BinCell {
    float2 mu;
    float2 md[8];
    int offx, offy;   // n_lo * (K + 1) per axis: bin = n * (K + 1) + sub - off
    int bx, by;       // bins per axis
    int base;         // first u32 counter of this cell in the warp's bin region
};

// Setup of cell c at layer t: error bound, envelope, bin box.  False when
// the cell cannot be binned (its f32 error exceeds the zone half-width, or
// its box is too large); the task then takes the per-transition path.
__device__ __forceinline__ bool bin_setup(const BuildK &K, int t, int c, BinCell &B, int &words)
{
    const size_t cell = (size_t)t * K.nc + c;
    const double2 mu = *reinterpret_cast<const double2 *>(K.mean + cell * 2);
    const double *cm = K.cmax + (size_t)(t - K.t0) * K.nm;
    const double ipz = 1.0 / K.bin_p;
    double Px = 0.0, Py = 0.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        B.md[m] = make_float2(0.f, 0.f);
        if (m < K.nm) {
            const double2 md = *reinterpret_cast<const double2 *>(K.modes + (((size_t)m * K.nt + t) * K.nc + c) * 2);
            // z = v / p directly: the modes and the mean carry 1/p (one
            // rounding of md / p to f32, the same 2^-24 relative as md alone)
            B.md[m] = make_float2((float)(md.x * ipz), (float)(md.y * ipz));
            const double w = cm[m];
            Px += fabs(md.x) * w;
            Py += fabs(md.y) * w;
        }
    }
    B.mu = make_float2((float)(mu.x * ipz), (float)(mu.y * ipz));
    const double Tx = fabs(mu.x) + Px, Ty = fabs(mu.y) + Py;
    // |v32 - v64| <= delta (the k_vmax bound: f32 inputs, FMA chain, and the
    // reference's own f64 rounding) -- here with the inputs pre-scaled by
    // 1/p, |z32 - v64 / p| <= delta / p + 2^-24 |v| / p; then floor/frac in
    // f32: 2^-21 (|z| + 1) covers that and the frac subtraction
    const double kRel = (2.0 * K.nm + 8.0) * 0x1p-24 * 1.001, kAbs = (K.nm + 2.0) * 0x1p-140;
    const double dlx = Tx * kRel + kAbs, dly = Ty * kRel + kAbs;
    const double ip = 1.0 / K.bin_p;
    const double Dx = dlx * ip + 0x1p-21 * (Tx * ip + 1.0) + K.bin_eps;
    const double Dy = dly * ip + 0x1p-21 * (Ty * ip + 1.0) + K.bin_eps;
    if (!(Dx <= K.bin_dzone && Dy <= K.bin_dzone)) return false;
    double xlo, xhi, ylo, yhi;
    if (K.envelope) {   // widened by delta in the scan: contains v64 and v32
        const int4 e = K.envelope[cell];
        xlo = ord_f32(e.x); xhi = ord_f32(e.y); ylo = ord_f32(e.z); yhi = ord_f32(e.w);
        xlo -= dlx; xhi += dlx; ylo -= dly; yhi += dly;
    } else {            // triangle bound around the mean
        xlo = mu.x - Px - 2.0 * dlx; xhi = mu.x + Px + 2.0 * dlx;
        ylo = mu.y - Py - 2.0 * dly; yhi = mu.y + Py + 2.0 * dly;
    }
    const double zxl = xlo * ip - Dx, zxh = xhi * ip + Dx, zyl = ylo * ip - Dy, zyh = yhi * ip + Dy;
    if (!(fabs(zxl) < 0x1p20 && fabs(zxh) < 0x1p20 && fabs(zyl) < 0x1p20 && fabs(zyh) < 0x1p20)) return false;
    const int nxl = (int)floor(zxl), nxh = (int)floor(zxh), nyl = (int)floor(zyl), nyh = (int)floor(zyh);
    B.bx = (nxh - nxl + 1) * K.bin_k1x;
    B.by = (nyh - nyl + 1) * K.bin_k1y;
    B.offx = nxl * K.bin_k1x;
    B.offy = nyl * K.bin_k1y;
    words = B.bx * B.by;
    return words <= K.bin_words;
}

// Exact f64 velocity of (t, r, cell c) in the reference's order
// (environment.py:293-297: v = mean; v = v + c_m * mode_m, ascending m).
__device__ __forceinline__ double2 exact_velocity(const BuildK &K, int t, int r, int c)
{
    const double2 mu = *reinterpret_cast<const double2 *>(K.mean + ((size_t)t * K.nc + c) * 2);
    double vx = mu.x, vy = mu.y;
    const double *cf = K.coeffs + ((size_t)t * K.nr + r) * K.nm;
    for (int m = 0; m < K.nm; ++m) {
        const double2 md = *reinterpret_cast<const double2 *>(K.modes + (((size_t)m * K.nt + t) * K.nc + c) * 2);
        const double k = __ldg(cf + m);
        vx = DADD(vx, DMUL(k, md.x));
        vy = DADD(vy, DMUL(k, md.y));
    }
    return make_double2(vx, vy);
}

// Deferred realizations of a lean bin task (within a zone, or out of the
// box): the exact f64 velocity, then every row of its cell takes the
// reference's transition (lean_transition, as the per-transition path) into
// the dense histogram.  Items are (cell slot << 16 | r); the last n <= 32
// are processed.
template <int FLAGS>
__device__ __forceinline__ int bin_drain(const BuildK &K, const uint32_t *bq, int qn, int t, int grp,
                                         const RowC &Rf, uint16_t *h16q, unsigned hs_word, int outq, bool row_ok,
                                         int cs_row, unsigned half_one, int &q_lo, int &q_hi)
{
    const int lane = threadIdx.x & 31;
    const int n = qn < 32 ? qn : 32, first = qn - n;
    if (lane == 0) FM_STAT(6, n);
    double2 v = make_double2(0.0, 0.0);
    int cs = -1;
    if (lane < n) {
        const uint32_t it = bq[first + lane];
        cs = (int)(it >> 16);
        v = exact_velocity(K, t, (int)(it & 0xFFFFu), K.cell0 + grp * K.CW + cs);
    }
    for (int e = 0; e < n; ++e) {
        const double vx = __shfl_sync(kFull, v.x, e), vy = __shfl_sync(kFull, v.y, e);
        const int ce = __shfl_sync(kFull, cs, e);
        if (row_ok && cs_row == ce) {
            double w;
            const int q = lean_transition<FLAGS, false>(K, Rf, make_double2(vx, vy), nullptr, outq, w);
            hist_inc(h16q, hs_word, q, half_one);
            if (q != outq) {
                q_lo = min(q_lo, q);
                q_hi = max(q_hi, q);
            }
        }
    }
    __syncwarp();
    return first;
}

// Obstacle bin tasks: queue items are (r | cell slot << 16 | kind), kind =
// bit 17 (a doubtful realization: not binned, every live row takes the
// exact transition) or the bin index << 18 (a binned realization whose bin
// marks, in its high half, the rows landing on a danger class 2 / 3 slot:
// those rows take the exact transit test and move the transition to OUT
// when it is blocked).  The work is spread over the warp per (item, row)
// pair; every dense-histogram update is a 32-bit shared-memory add on the
// word holding the owner row's u16 counter (+-1 << 16 * (owner & 1)), so
// the pairs' +-1 and the epilogue's rectangle sums commute modulo 2^32 and
// the final halves are exact (each true count lies in [0, 65535]).
// environment.py:338-368 (transit test), model_builder.py:331-347 (landing).
static constexpr uint32_t kItemD = 1u << 17;
struct ObstDrainBuf {
    double2 v[32];
    int32_t scan[32];
    uint32_t mask[32];
    uint32_t meta[32];
    // per task: the cells' centres (environment.py:99-100), columns / rows,
    // window offsets, and the task's action vectors
    double2 x0[2];
    int32_t ci[2], cj[2], soff[2], pad_[2];
    double2 act[32];
};

template <int FLAGS>
__device__ __noinline__ int bin_drain_obst(const BuildK &K, const uint32_t *bq, const uint32_t *bins, int qn, int t,
                                              int grp, int ag, unsigned dense_s, const uint32_t *danger, int CWD,
                                              ObstDrainBuf *db, const double *ftab_s, const uint8_t *mwin)
{
    const int ww = 2 * K.hx + 3, wh = 2 * K.hy + 3;
    const int lane = threadIdx.x & 31;
    const int n = qn < 32 ? qn : 32, first = qn - n;
    if (lane == 0) FM_STAT(6, n);
    const int AG = K.AG;
    const int na_loc = min(AG, K.na - ag * 32);
    int cnt = 0;
#ifdef FM_STATS
    const unsigned gw = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % (148 * 64);
    if (lane < n) atomicAdd(&g_fm_wcnt[gw][(bq[first + lane] & kItemD) ? 0 : 1], 1u);
#endif
    if (lane < n) {
        const uint32_t it = bq[first + lane];
        const int cs = (int)((it >> 16) & 1u);
        const int r = (int)(it & 0xFFFFu);
        db->v[lane] = exact_velocity(K, t, r, K.cell0 + grp * K.CW + cs);
        const uint32_t m = (it & kItemD) ? (na_loc >= 32 ? 0xFFFFFFFFu : (1u << na_loc) - 1u) : (bins[it >> 18] >> 16);
        db->mask[lane] = m;
        db->meta[lane] = it;
        cnt = __popc(m);
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    db->scan[lane] = incl;
    const int total = __shfl_sync(kFull, incl, 31);
    __syncwarp();
#ifdef FM_STATS
    const long long cp0 = clock64();
#endif
    for (int k = lane; k < total; k += 32) {
        // item e: the first with scan[e] > k; row: the j-th set bit of its mask
        int lo = 0, hi = n - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (db->scan[mid] > k) hi = mid;
            else lo = mid + 1;
        }
        const int e = lo;
        const int j = k - (e ? db->scan[e - 1] : 0);
        unsigned al;
        asm("fns.b32 %0, %1, 0, %2;" : "=r"(al) : "r"(db->mask[e]), "r"(j + 1));
        const uint32_t it = db->meta[e];
        const int cs = (int)((it >> 16) & 1u);
        const int owner = cs * AG + (int)al;
        // the row's constants (model_builder.py:331-335), staged per task
        RowC R;
        R.ci = db->ci[cs];
        R.cj = db->cj[cs];
        R.x0 = db->x0[cs].x;
        R.y0 = db->x0[cs].y;
        R.ax = db->act[al].x;
        R.ay = db->act[al].y;
        R.soff = db->soff[cs];
        const uint32_t *cls = danger + cs * CWD;
        const double2 v = db->v[e];
        double px = DADD(v.x, R.ax), py = DADD(v.y, R.ay);   // x' = x0 + (v + a) * dt
        if (!(FLAGS & F_DT_ONE)) {
            px = DMUL(px, K.dt);
            py = DMUL(py, K.dt);
        }
        const double x1 = DADD(R.x0, px), y1 = DADD(R.y0, py);
        const int i1 = floor_magic(to_cell<FLAGS>(x1, K.ox, K.dx, K.inv_dx));
        const int j1 = floor_magic(to_cell<FLAGS>(y1, K.oy, K.dx, K.inv_dx));
        const int slot = j1 * K.width + i1 + R.soff;   // inside the window (F_PROVEN)
        const int cl = (int)((cls[slot >> 4] >> ((slot & 15) << 1)) & 3u);
#ifdef FM_STATS
        atomicAdd(&g_fm_wcnt[gw][2], 1u);
        if (cl >= 2) atomicAdd(&g_fm_wcnt[gw][3], 1u);
#endif
        const bool blocked = cl >= 2 && !(K.dev_flags & 1) && seg_samples_blocked_win<FLAGS>(K, ftab_s, mwin + cs * ww * wh,
                                                                      R.ci - K.hx - 1, R.cj - K.hy - 1, ww, wh, t,
                                                                      R.x0, R.y0, x1, y1);
        const unsigned sh = (unsigned)(owner & 1) * 16u;
        const unsigned wofs = (unsigned)(owner >> 1) * 4u;
        const unsigned w_slot = dense_s + (unsigned)slot * 64u + wofs;
        const unsigned w_out = dense_s + (unsigned)K.nslot * 64u + wofs;
        if (it & kItemD) {   // not binned: the whole transition here
            const unsigned w = (cl == 1 || blocked) ? w_out : w_slot;
            asm volatile("red.shared.add.u32 [%0], %1;\n" ::"r"(w), "r"(1u << sh) : "memory");
        } else if (blocked) {   // binned in its landing slot: move it to OUT
            asm volatile("red.shared.add.u32 [%0], %1;\n" ::"r"(w_slot), "r"(0u - (1u << sh)) : "memory");
            asm volatile("red.shared.add.u32 [%0], %1;\n" ::"r"(w_out), "r"(1u << sh) : "memory");
        }
    }
    __syncwarp();
#ifdef FM_STATS
    if (lane == 0) g_fm_wcnt[gw][7] += (unsigned)((clock64() - cp0) >> 6);
#endif
    return first;
}

// The realization loop of one bin task over NC (1 or 2) cells: f32
// reconstruction, bin, one shared-memory increment per (cell, realization);
// realizations with any doubt are queued for the exact path.  Coefficients
// stream through a per-warp ring of 32-realization chunks (cp.async, RING
// chunks in flight), two chunks per iteration.  Lean tasks (OB = false):
// returns the queue length, or -1 when the queue overflowed (the task then
// takes the per-transition path).  Obstacle tasks (OB = true): a bin's high
// half holds the mask of the rows whose landing from it lies on a danger
// class 2 / 3 slot (set by bin_task); a realization binned there is counted
// and also queued (the atomic returns the bin's old value), and the queue
// is drained (`drain`, bin_drain_obst) whenever the next iteration could
// overflow it.
#ifndef FM_BIN_H
#define FM_BIN_H 2
#endif
template <int NC, bool OB, int RING, typename Drain>
__device__ __forceinline__ int bin_loop(const BuildK &K, const BinCell *B, const int *cid, bool two, int t,
                                        const BinEnt *tab_s, unsigned bins_s, unsigned ring_s, uint32_t *bq,
                                        Drain &&drain)
{
    const int lane = threadIdx.x & 31, nr = K.nr;
    const int nch = K.nr_pad >> 5;   // a multiple of H: coefficients zero-padded to whole iterations
    const float2 M2 = make_float2(12582912.0f, 12582912.0f);   // 1.5 * 2^23: floor by a round-down add
    const int ns = K.bin_ns;
    const float2 NS2 = make_float2((float)ns, (float)ns);
    // bucket bits -> this lane's copy of the table entry ([axis][bucket][copy]
    // of 8 B: lanes l and l + 16 share a copy, so a lookup is conflict-free):
    // one opaque base with the bias folded in
    unsigned tabx_s;
    asm("mov.b32 %0, %1;"
        : "=r"(tabx_s)
        : "r"((unsigned)__cvta_generic_to_shared(tab_s) + 8u * (unsigned)(lane & (kBinRep - 1)) -
              0x4B400000u * (8u * kBinRep)));
    const unsigned taby_s = tabx_s + (unsigned)(ns + 1) * (8u * kBinRep);
    const int k1x = K.bin_k1x, k1y = K.bin_k1y;
    constexpr int QCAP = OB ? kBinQO : kBinQ;
    // bin = (bits(M + floor z) - bits(M)) * k1 + kb - off, with kb + 1 in the
    // table entry's low bits: the -1, the bias and the offset fold into one
    // constant (modulo 2^32: the products with the bias bits wrap and cancel)
    unsigned cx[NC], cy[NC];
    unsigned bxn[NC], byn[NC];
    unsigned bb[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        cx[q] = 0u - 0x4B400000u * (unsigned)k1x - (unsigned)B[q].offx - 1u;
        cy[q] = 0u - 0x4B400000u * (unsigned)k1y - (unsigned)B[q].offy - 1u;
        bxn[q] = (unsigned)B[q].bx;
        byn[q] = (unsigned)B[q].by;
        bb[q] = bins_s + 4u * (unsigned)B[q].base;
    }
    // realizations that are not counted (doubtful, or padding) add to a
    // per-lane dummy counter past the task's bins: no branch per update
    const unsigned dummy = bins_s + 4u * (unsigned)(K.bin_words - 32 + lane);
    const char *gsrc = reinterpret_cast<const char *>(K.coef32 + (size_t)(t - K.t0) * K.nr_pad * 8 + lane * 8);
    // a ring chunk (32 realizations x 8 f32): [coefficients 0-3 of the 32
    // lanes | coefficients 4-7]: each 16-byte lane read is conflict-free
    const unsigned rl = ring_s + (unsigned)lane * 16u;
    auto issue = [&](int i) {
        if (i < nch) {
            const unsigned d = rl + (unsigned)(i & (RING - 1)) * 1024u;
            const char *src = gsrc + (size_t)i * 1024;
            // .ca: the warps of an SM sweep the same slab's coefficients
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d + 512u), "l"(src + 16) : "memory");
        }
        cp_async_commit();
    };
#pragma unroll
    for (int i = 0; i < RING - ((RING >= 8) ? FM_BIN_H : 2); ++i) issue(i);
    int qn = 0;
    constexpr int H = (RING >= 8) ? FM_BIN_H : 2;   // chunks (of 32 realizations) per iteration
    {
        for (int i = 0; i < nch; i += H) {
#pragma unroll
            for (int h = 0; h < H; ++h) issue(i + RING - H + h);
            asm volatile("cp.async.wait_group %0;\n" ::"n"(RING - H) : "memory");
            __syncwarp();
            bool dq[H][NC];
            uint32_t it_[H][NC];
            // both chunks' coefficients first (volatile: behind the cp.async
            // wait, and ahead of every counter update so the two chunks'
            // chains interleave; the table loads below are plain -- the
            // tables never change during the loop)
            float4 c0[H], c1[H];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const unsigned ra = rl + (unsigned)((i + h) & (RING - 1)) * 1024u;
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(c0[h].x), "=f"(c0[h].y), "=f"(c0[h].z), "=f"(c0[h].w) : "r"(ra));
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(c1[h].x), "=f"(c1[h].y), "=f"(c1[h].z), "=f"(c1[h].w) : "r"(ra + 512u));
            }
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const int r = (i + h) * 32 + lane;
                const bool live_r = r < nr;   // padded realizations (zero coefficients) are binned, never counted
                const float cf[8] = {c0[h].x, c0[h].y, c0[h].z, c0[h].w, c1[h].x, c1[h].y, c1[h].z, c1[h].w};
#pragma unroll
                for (int q = 0; q < NC; ++q) {
                    const bool live = live_r && (q == 0 || two);
                    // (one chain: two interleaved half-chains + an add measured slower)
                    float2 v = B[q].mu;
#pragma unroll
                    for (int m = 0; m < 8; ++m) v = ffma2_bcast(cf[m], B[q].md[m], v);
                    const float2 z = v;   // the inputs carry 1/p (bin_setup)
                    const float2 t1 = f2_add_rm(z, M2);             // M + floor(z)
                    const float2 f = f2_sub(z, f2_sub(t1, M2));     // frac(z) in [0, 1] (z finite: F_PROVEN)
                    const float2 tb = f2_fma_rm(f, NS2, M2);        // M + floor(frac * NS), <= M + NS
                    float2 ex, ey;   // (lo | kb + 1 in the low mantissa bits, hi)
                    asm("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(ex.x), "=f"(ex.y) : "r"(tabx_s + (8u * kBinRep) * (unsigned)__float_as_int(tb.x)));
                    asm("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(ey.x), "=f"(ey.y) : "r"(taby_s + (8u * kBinRep) * (unsigned)__float_as_int(tb.y)));
                    // sign bits: f < lo (below the zone), f > hi (above it)
#ifndef FM_ZONE_PACKED
                    // scalar subtractions: no register moves to pair the table halves
                    float2 dlo, dhi;
                    asm("sub.rn.f32 %0, %1, %2;" : "=f"(dlo.x) : "f"(f.x), "f"(ex.x));
                    asm("sub.rn.f32 %0, %1, %2;" : "=f"(dlo.y) : "f"(f.y), "f"(ey.x));
                    asm("sub.rn.f32 %0, %1, %2;" : "=f"(dhi.x) : "f"(ex.y), "f"(f.x));
                    asm("sub.rn.f32 %0, %1, %2;" : "=f"(dhi.y) : "f"(ey.y), "f"(f.y));
#else
                    const float2 dlo = f2_sub(f, make_float2(ex.x, ey.x));
                    const float2 dhi = f2_sub(make_float2(ex.y, ey.y), f);
#endif
                    const unsigned sx = (unsigned)__float_as_int(dhi.x) >> 31, sy = (unsigned)__float_as_int(dhi.y) >> 31;
                    const unsigned bx = (unsigned)__float_as_int(t1.x) * (unsigned)k1x + cx[q] +
                                        ((unsigned)__float_as_int(ex.x) & 63u) + sx;
                    const unsigned by = (unsigned)__float_as_int(t1.y) * (unsigned)k1y + cy[q] +
                                        ((unsigned)__float_as_int(ey.x) & 63u) + sy;
                    // safe: outside this bucket's zone on both axes and inside the box
                    const unsigned zs = ((unsigned)__float_as_int(dlo.x) | (unsigned)__float_as_int(dhi.x)) &
                                        ((unsigned)__float_as_int(dlo.y) | (unsigned)__float_as_int(dhi.y));
                    const bool ok = live & ((zs >> 31) != 0u) & (bx < bxn[q]) & (by < byn[q]);
                    const unsigned widx = by * bxn[q] + bx;
                    const unsigned addr = ok ? bb[q] + 4u * widx : dummy;
                    uint32_t item = kItemD;
                    bool gated = false;
                    if (OB) {   // counted either way; a bin with a row mask also queues it
                        unsigned old;
                        asm volatile("atom.shared.add.u32 %0, [%1], 1;\n" : "=r"(old) : "r"(addr) : "memory");
                        gated = ok & ((old >> 16) != 0u);
                        if (ok) item = (uint32_t)(B[q].base + (int)widx) << 18;
                    } else {   // no memory clobber: the callers fence before reading the bins
                        asm volatile("red.shared.add.u32 [%0], 1;\n" ::"r"(addr));
                    }
                    dq[h][q] = live & (!ok | gated);
                    it_[h][q] = item | ((uint32_t)cid[q] << 16) | (uint32_t)r;
                }
            }
            bool any = false;
#pragma unroll
            for (int h = 0; h < H; ++h)
#pragma unroll
                for (int q = 0; q < NC; ++q) any |= dq[h][q];
            if (__any_sync(kFull, any)) {
#pragma unroll
                for (int h = 0; h < H; ++h)
#pragma unroll
                    for (int q = 0; q < NC; ++q) {
                        const unsigned bm = __ballot_sync(kFull, dq[h][q]);
                        const int pos = qn + __popc(bm & ((1u << lane) - 1u));
                        if (dq[h][q] && pos < QCAP) bq[pos] = OB ? it_[h][q] : (((uint32_t)cid[q] << 16) | (uint32_t)((i + h) * 32 + lane));
                        qn += __popc(bm);
                    }
                if (OB) {
                    if (qn > QCAP - H * NC * 32) {   // the next iteration could overflow: drain now
                        __syncwarp();
                        drain(qn);
                        qn = 0;
                    }
                } else if (qn > QCAP) {   // too many doubtful realizations: per transition instead
                    cp_async_wait_all();
                    __syncwarp();
                    return -1;
                }
            }
            __syncwarp();
        }
    }
    cp_async_wait_all();
    __syncwarp();
    return qn;
}

__device__ __forceinline__ int floordiv_pos(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// A task by binning (see the comment at kBinNS).  Lean tasks (OB = false)
// and, under F_PROVEN | F_CNT, obstacle tasks (OB = true: dead cells count
// nothing, landings on a cell masked at t+1 go to OUT in the epilogue, and
// every realization from which some action's landing slot needs the exact
// transit test -- danger class 2 / 3 -- takes the exact path for all its
// rows).  Returns false when some cell cannot be binned or (lean) too many
// realizations need the exact path; the caller then runs the per-transition
// path (which clears its own histogram).  On success the task's dense
// [slot][row] histogram at wbase + off_bdense holds exactly the counts the
// per-transition path would produce.
template <int FLAGS, bool OB>
__device__ __forceinline__ bool bin_task(const BuildK *__restrict__ Kg, unsigned char *wbase, const BinEnt *tab_s, int t,
                                         int grp, int ag, const RowC &Rf, int outq, bool row_ok, int cs_row,
                                         unsigned half_one, const uint32_t *danger, int &q_lo, int &q_hi)
{
    const BuildK &K = *Kg;
    const int lane = threadIdx.x & 31;
    const int CW = K.CW;
    const int CWD = 2 * ((K.nslot + 31) >> 5);   // danger-map words per cell
    // cells of the task that bin (obstacle tasks: dead cells -- the target,
    // obstacle cells at t -- send every realization to OUT, model_builder.py:445-452)
    auto cell_live = [&](int cs) {
        const int lc = grp * CW + cs;
        if (cs >= CW || lc >= K.ncell) return false;
        if (OB) {
            const int c = K.cell0 + lc;
            if (c == K.tcell || K.mask[(size_t)t * K.nc + c]) return false;
        }
        return true;
    };
    if (OB && K.AG > 16) return false;   // the row masks take a bin's high half
    // every cell must fit before anything is written
    for (int p = 0; p < CW; p += 2) {
        int words = 0;
        for (int q = 0; q < 2; ++q) {
            if (cell_live(p + q)) {
                BinCell B;
                int w;
                if (!bin_setup(K, t, K.cell0 + grp * CW + p + q, B, w)) return false;
                words += w;
            }
        }
        if (words > K.bin_words - 32) return false;   // + 32 per-lane dummy counters (bin_loop)
    }
    uint32_t *bins = reinterpret_cast<uint32_t *>(wbase + K.off_bins);
    uint32_t *bq = reinterpret_cast<uint32_t *>(wbase + K.off_bq);
    const unsigned bins_s = (unsigned)__cvta_generic_to_shared(bins);
    const unsigned ring_s = (unsigned)__cvta_generic_to_shared(wbase + K.off_bring);
    uint16_t *h16 = reinterpret_cast<uint16_t *>(wbase + K.off_bdense) + lane;
    uint16_t *h16q = h16 + Rf.soff * 32;
    const unsigned hs_word = (unsigned)__cvta_generic_to_shared(h16q) & ~3u;
    const int k1x = K.bin_k1x, k1y = K.bin_k1y;
    const int a = ag * 32 + (lane - cs_row * K.AG);
    const uint32_t *cls_row = danger + cs_row * CWD;
    const bool live_row = row_ok && (!OB || !(Rf.rflags & RF_DEAD));
    const unsigned dense_s = (unsigned)__cvta_generic_to_shared(wbase + K.off_bdense);
    ObstDrainBuf *db = reinterpret_cast<ObstDrainBuf *>(wbase + K.off_bq + kBinQO * 4);
    uint8_t *mwin = reinterpret_cast<uint8_t *>(db + 1);   // [CW][2hy + 3][2hx + 3] mask at t
    const double *ftab_s = reinterpret_cast<const double *>(tab_s + 2 * (K.bin_ns + 1) * kBinRep);
    auto drain_all = [&](int qn) {
#ifdef FM_STATS
        const long long c0 = clock64();
#endif
        for (int n = qn; n > 0;) {
            if (OB) n = bin_drain_obst<FLAGS>(K, bq, bins, n, t, grp, ag, dense_s, danger, CWD, db, ftab_s, mwin);
            else n = bin_drain<FLAGS>(K, bq, n, t, grp, Rf, h16q, hs_word, outq, live_row, cs_row, half_one, q_lo, q_hi);
        }
#ifdef FM_STATS
        if (OB && lane == 0)
            g_fm_wcnt[(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % (148 * 64)][5] += (unsigned)((clock64() - c0) >> 6);
#endif
    };
    if (OB) {   // the ring sits beside the dense histogram: zero it up front (mid-loop drains)
        for (int sl = 0; sl <= K.nslot; ++sl) h16[sl * 32] = 0;
        const int ww = 2 * K.hx + 3, wh = 2 * K.hy + 3;
        if (lane < CW) {
            const int c = K.cell0 + grp * CW + lane, ci = c % K.nx, cj = c / K.nx;
            db->ci[lane] = ci;
            db->cj[lane] = cj;
            db->x0[lane] = make_double2(DADD(K.ox, DMUL(DADD((double)ci, 0.5), K.dx)),
                                        DADD(K.oy, DMUL(DADD((double)cj, 0.5), K.dx)));
            db->soff[lane] = -((cj - K.hy) * K.width + (ci - K.hx));
        }
        if (lane < min(K.AG, K.na - ag * 32)) {
            const fm_action A = K.act[ag * 32 + lane];
            db->act[lane] = make_double2(A.ax, A.ay);
        }
        for (int cs = 0; cs < CW; ++cs) {
            if (!cell_live(cs)) continue;
            const int c = K.cell0 + grp * CW + cs, i0 = c % K.nx - K.hx - 1, j0 = c / K.nx - K.hy - 1;
            for (int k = lane; k < ww * wh; k += 32) {
                const int i = i0 + k % ww, j = j0 + k / ww;
                mwin[cs * ww * wh + k] =
                    ((unsigned)i < (unsigned)K.nx && (unsigned)j < (unsigned)K.ny) ? K.mask[(size_t)t * K.nc + j * K.nx + i] : 0;
            }
        }
        __syncwarp();
    }
    for (int p = 0; p < CW; p += 2) {
        // the pair's live cells, compacted (constant indices keep B in registers)
        const bool l0 = cell_live(p), l1 = cell_live(p + 1);
        const bool two = l0 && l1;
        const int ncl = (l0 ? 1 : 0) + (l1 ? 1 : 0);
        const int cid[2] = {l0 ? p : p + 1, p + 1};
        BinCell B[2];
        int words = 0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            int w = 0;
            if (q < ncl) {
                bin_setup(K, t, K.cell0 + grp * CW + cid[q], B[q], w);
            } else {   // a missing cell still runs through the loop: finite inputs (table indices)
                B[q].bx = B[q].by = B[q].offx = B[q].offy = 0;
                B[q].mu = make_float2(0.f, 0.f);
#pragma unroll
                for (int m = 0; m < 8; ++m) B[q].md[m] = make_float2(0.f, 0.f);
            }
            B[q].base = words;
            words += w;
        }
#ifdef FM_STATS
        const long long ci0 = clock64();
#endif
        if (OB) {
            // high half of each bin: the rows (task-local actions) whose
            // landing from it lies on a slot of class 2 / 3 (the tight or
            // grown box touches the mask at t: exact transit test)
            const int na_loc = min(K.AG, K.na - ag * 32);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (q >= ncl) continue;
                const uint32_t *cl = danger + cid[q] * CWD;
                bool anyg = false;
                for (int i = 0; i < CWD; ++i) anyg |= (cl[i] & 0xAAAAAAAAu) != 0u;
                uint32_t *b = bins + B[q].base;
                const int bxn = B[q].bx, nw = B[q].bx * B[q].by;
                for (int w = lane; w < nw; w += 32) {
                    uint32_t g = 0u;
                    if (anyg) {
                        const int by = w / bxn, bx = w - by * bxn;
                        const int bax = bx + B[q].offx, bay = by + B[q].offy;
                        const int nxv = floordiv_pos(bax, k1x), sxv = bax - nxv * k1x;
                        const int nyv = floordiv_pos(bay, k1y), syv = bay - nyv * k1y;
                        for (int al = 0; al < na_loc; ++al) {
                            const BinAct ba = K.bact[ag * 32 + al];
                            const int di = ba.gx + nxv + (sxv >= ba.rx ? 1 : 0);
                            const int dj = ba.gy + nyv + (syv >= ba.ry ? 1 : 0);
                            if ((unsigned)(di + K.hx) <= (unsigned)(2 * K.hx) &&
                                (unsigned)(dj + K.hy) <= (unsigned)(2 * K.hy)) {
                                const int slot = (dj + K.hy) * K.width + di + K.hx;
                                if ((cl[slot >> 4] >> ((slot & 15) << 1)) & 2u) g |= 1u << al;
                            }
                        }
                    }
                    b[w] = g << 16;
                }
            }
        } else {
            for (int w = lane; w < words; w += 32) bins[w] = 0u;
        }
        __syncwarp();
#ifdef FM_STATS
        const long long ci1 = clock64();
        if (OB && lane == 0) g_fm_wcnt[(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % (148 * 64)][4] += (unsigned)((ci1 - ci0) >> 6);
#endif
        int qn = 0;
        constexpr int RING = OB ? kBinRingO : kBinRing;
        // one loop instance (code size): a missing second cell never counts
        // a lean pair with one live cell (|A| > 16: one cell per task) runs
        // the one-cell instance -- half the reconstructions and counter
        // updates of the pair loop, which would compute a dead second cell
        if constexpr (!OB) {
            if (ncl == 1) qn = bin_loop<1, OB, RING>(K, B, cid, false, t, tab_s, bins_s, ring_s, bq, drain_all);
            else if (ncl > 1) qn = bin_loop<2, OB, RING>(K, B, cid, two, t, tab_s, bins_s, ring_s, bq, drain_all);
        } else {
            if (ncl > 0) qn = bin_loop<2, OB, RING>(K, B, cid, two, t, tab_s, bins_s, ring_s, bq, drain_all);
        }
        if (qn < 0) return false;
        FM_STAT(5, lane == 0 ? 1 : 0);
#ifdef FM_STATS
        if (OB && lane == 0) g_fm_wcnt[(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % (148 * 64)][6] += (unsigned)((clock64() - ci1) >> 6);
#endif
        // lean tasks: the ring is done, its space becomes the dense histogram
        // (zeroed once, at the first pair); then the deferred realizations
        if (!OB && p == 0) {
            for (int sl = 0; sl <= K.nslot; ++sl) h16[sl * 32] = 0;
            __syncwarp();
        }
        drain_all(qn);
        asm volatile("" ::: "memory");
        __syncwarp();
        if (OB) {   // drop the row masks: the low halves are the counts
            for (int w = lane; w < words; w += 32) bins[w] &= 0xFFFFu;
            __syncwarp();
        }
        // 2-D inclusive prefix sums of each cell's bins (rows, then columns)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            uint32_t *b = bins + B[q].base;
            for (int y = lane; y < B[q].by; y += 32) {
                uint32_t acc = 0;
                for (int x = 0; x < B[q].bx; ++x) {
                    acc += b[y * B[q].bx + x];
                    b[y * B[q].bx + x] = acc;
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            uint32_t *b = bins + B[q].base;
            for (int x = lane; x < B[q].bx; x += 32) {
                uint32_t acc = 0;
                for (int y = 0; y < B[q].by; ++y) {
                    acc += b[y * B[q].bx + x];
                    b[y * B[q].bx + x] = acc;
                }
            }
        }
        __syncwarp();
        // each row: its (di, dj) counts are rectangle sums over the bins
        if (live_row && ncl > 0 && (cs_row == cid[0] || (two && cs_row == cid[1]))) {
            // the row's cell (selects keep B in registers: no dynamic index)
            const bool q1 = two && cs_row == cid[1];
            const int offx = q1 ? B[1].offx : B[0].offx, offy = q1 ? B[1].offy : B[0].offy;
            const int cbx = q1 ? B[1].bx : B[0].bx, cby = q1 ? B[1].by : B[0].by;
            const uint32_t *b = bins + (q1 ? B[1].base : B[0].base);
            const BinAct ba = K.bact[a];
            const int nxl = offx / k1x, nxh = nxl + cbx / k1x - 1;
            const int nyl = offy / k1y, nyh = nyl + cby / k1y - 1;
            const int dil = ba.gx + nxl + (ba.rx == 0 ? 1 : 0), dih = ba.gx + nxh + (ba.rx <= k1x - 1 ? 1 : 0);
            const int djl = ba.gy + nyl + (ba.ry == 0 ? 1 : 0), djh = ba.gy + nyh + (ba.ry <= k1y - 1 ? 1 : 0);
            for (int dj = djl; dj <= djh; ++dj) {
                const int ey = dj - ba.gy;
                const int y0 = max((ey - 1) * k1y + ba.ry - offy, 0);
                const int y1 = min(ey * k1y + ba.ry - 1 - offy, cby - 1);
                if (y0 > y1) continue;
                for (int di = dil; di <= dih; ++di) {
                    const int ex = di - ba.gx;
                    const int x0 = max((ex - 1) * k1x + ba.rx - offx, 0);
                    const int x1 = min(ex * k1x + ba.rx - 1 - offx, cbx - 1);
                    if (x0 > x1) continue;
                    uint32_t cnt = b[y1 * cbx + x1];
                    if (x0 > 0) cnt -= b[y1 * cbx + x0 - 1];
                    if (y0 > 0) cnt -= b[(y0 - 1) * cbx + x1];
                    if (x0 > 0 && y0 > 0) cnt += b[(y0 - 1) * cbx + x0 - 1];
                    if (cnt) {
                        // inside the window by the F_PROVEN proof
                        if ((unsigned)(di + K.hx) <= (unsigned)(2 * K.hx) && (unsigned)(dj + K.hy) <= (unsigned)(2 * K.hy)) {
                            int qq = (Rf.cj + dj) * K.width + (Rf.ci + di);
                            if (OB) {
                                // class 1: the landing cell is masked at t+1 -> OUT;
                                // a 32-bit add (see bin_drain_obst)
                                const int slot = qq + Rf.soff;
                                if (((cls_row[slot >> 4] >> ((slot & 15) << 1)) & 3u) == 1u) qq = outq;
                                asm volatile("red.shared.add.u32 [%0], %1;\n" ::"r"(hs_word + (unsigned)qq * 64u),
                                             "r"(half_one * cnt)
                                             : "memory");
                            } else {
                                h16q[qq * 32] += (uint16_t)cnt;
                                q_lo = min(q_lo, qq);
                                q_hi = max(q_hi, qq);
                            }
                        } else {
                            atomicOr(K.viol + (size_t)t * K.na + a, 2u);   // cannot happen: flags a bug loudly
                        }
                    }
                }
            }
        }
        __syncwarp();
    }
    return true;
}

// One warp = one task (t, group of CW source cells, group of <=32 actions).
// Lane roles:
//   row lane  (cs, a): owns the row (state t*N_c + c, action a); walks the
//                      realizations in ascending order, so its reward sum is
//                      the reference's sequential sum (model_builder.py:457);
//                      its displacement histogram (u16 counters, two per
//                      word, lane-interleaved -> conflict-free) lives in smem.
//   recon lane (cs, rr): reconstructs v(t, c, r) for a chunk of RW
//                      realizations into smem (environment.py:293-297), shared
//                      by all AG row lanes of that cell.  Coefficients of the
//                      next chunk stream in with cp.async while the row lanes
//                      work on the current one.
//
// PART splits the tasks by warp class so each launch carries only the code
// its warps run (the full kernel's instruction footprint thrashes the
// instruction cache: ncu "no instruction" stalls):
//   0 all tasks, 1 tasks without obstacle / dead rows (lean code only),
//   2 the rest.  Both parts classify every task the same way and skip the
//   other part's tasks.
#ifndef FM_BUILD_MINB
#define FM_BUILD_MINB 4
#endif
static_assert(FM_BUILD_RC <= 64, "chunk_rows_obst_cnt marks deferred realizations in a 64-bit mask");
#ifndef FM_BUILD_MINB1
#define FM_BUILD_MINB1 3
#endif
// PART 3 / 4: lean / obstacle tasks by binning only (bin_task); a task that
// cannot bin is appended to K.task_list and run by a PART 0 launch over the
// list, so these launches carry no per-transition code (instruction cache).
#ifndef FM_BUILD_MINB3
#define FM_BUILD_MINB3 4   // lean bin-only launch: 16 warps / SM (128 registers, no spills)
#endif
template <int FLAGS, int PART>
__global__ void __launch_bounds__(128, PART == 3 ? FM_BUILD_MINB3
                                      : (PART != 0 && (FLAGS & F_PROVEN) && (FLAGS & F_CNT)) ? FM_BUILD_MINB1
                                                                                              : FM_BUILD_MINB)
    k_build(const __grid_constant__ BuildK K)
{
    constexpr bool OBST_PART = PART == 2 || PART == 4, LEAN_PART = PART == 1 || PART == 3, BINONLY = PART >= 3;
    const BuildK *__restrict__ Kg = &K;   // the parameter block, for the noinline rare paths
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *wbase = smem + K.off_block + (size_t)warp * K.smem_warp;
    // bin tables (lean tasks binned per realization): block-shared copy
    const BinEnt *tab_s = reinterpret_cast<const BinEnt *>(smem);
    if constexpr (PART != 0 && (FLAGS & F_PROVEN) && (FLAGS & F_CNT)) {
        if (K.bin_ok) {
            BinEnt *t_s = reinterpret_cast<BinEnt *>(smem);   // [axis][bucket][kBinRep copies]
            const int per_axis = (K.bin_ns + 1) * kBinRep;
            for (int i = threadIdx.x; i < 2 * per_axis; i += blockDim.x) {
                const int ax = i / per_axis, bkt = (i - ax * per_axis) / kBinRep;
                t_s[i] = K.tab[ax * (kBinNS + 1) + bkt];
            }
            if (OBST_PART) {
                double *f_s = reinterpret_cast<double *>(t_s + 2 * per_axis);
                for (int i = threadIdx.x; i < (kFracSmemN + 1) * (kFracSmemN + 2) / 2; i += blockDim.x) f_s[i] = g_frac[i];
            }
            __syncthreads();
        }
    }
    uint16_t *hist16 = (FLAGS & F_GHIST)                                     // [nslot+1][32]
                           ? K.ghist + ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * (size_t)(K.nslot + 1) * 32
                           : reinterpret_cast<uint16_t *>(wbase);
    uint16_t *h16 = hist16 + lane;   // the task's dense histogram (a binned task moves it: bin_task)
    double2 *vbuf = reinterpret_cast<double2 *>(wbase + K.off_vbuf);       // [CW][RC+1]
    double *coefT = reinterpret_cast<double *>(wbase + K.off_coef);        // [nm][RC]
    double2 *modes_s = reinterpret_cast<double2 *>(wbase + K.off_modes);   // [CW][nm]
    uint32_t *danger = reinterpret_cast<uint32_t *>(wbase + K.off_danger);  // [CW][ceil(nslot/32)]

    for (int sl = 0; sl <= K.nslot; ++sl) h16[sl * 32] = 0;

    const int AG = K.AG, RW = K.RW, CW = K.CW, nm = K.nm, nr = K.nr;
    const int RC = K.RC, RPL = (RC + RW - 1) / RW;   // RW need not divide RC (e.g. |A| = 6: RW = 6)
    const int cs_row = lane / AG, a_loc = lane - cs_row * AG;
    const bool row_lane = lane < CW * AG;
    const int cs_rec = lane / RW, rr = lane - cs_rec * RW;
    const bool rec_lane = lane < CW * RW;
    const int nslot = K.nslot, W = K.width;
    const unsigned half_one = 1u << ((lane & 1) * 16);   // this lane's u16 half of a counter word
    // this lane's first (realization, mode) element of a coefficient chunk and
    // the per-step increments (element index advances by 32 each step)
    const int e_r0 = nm ? lane / nm : 0, e_m0 = nm ? lane - (lane / nm) * nm : 0;
    const int e_dr = nm ? 32 / nm : 0, e_dm = nm ? 32 - (32 / nm) * nm : 0;
    // same for the paired (16-byte) layout: element = (realization, mode pair)
    const int np2 = nm >> 1;
    const int p_r0 = np2 ? lane / np2 : 0, p_p0 = np2 ? lane - (lane / np2) * np2 : 0;
    const int p_dr = np2 ? 32 / np2 : 0, p_dp = np2 ? 32 - (32 / np2) * np2 : 0;

    for (;;) {
        unsigned task = 0;
        if (lane == 0) task = atomicAdd(K.task_counter, 1u);
        task = __shfl_sync(kFull, task, 0);
        if (PART == 0 && K.task_list) {   // the tasks the bin-only launches could not bin
            if (task >= *K.task_list_n) break;
            task = K.task_list[task];
        } else if (BINONLY) {   // this launch's classified tasks
            const unsigned na_ = *K.src_a_n;
            if (task < na_) {
                task = K.src_a[task];
            } else {
                task -= na_;
                if (!K.src_b || task >= *K.src_b_n) break;
                task = K.src_b[task];
            }
        } else if ((long long)task >= K.n_tasks) {
            break;
        }
#ifdef FM_STATS
        const long long tclk0 = clock64();
        int tpath = 0;
#endif
        h16 = hist16 + lane;
        const int per_t = K.groups * K.nag;
        const int t = K.t0 + (int)(task / per_t);
        const int rem = (int)(task % per_t);
        const int grp = rem / K.nag, ag = rem - (rem / K.nag) * K.nag;
        const int a = ag * 32 + a_loc;
        const int lc_row = grp * CW + cs_row;
        const bool row_ok = row_lane && lc_row < K.ncell && a < K.na;
        const int c = K.cell0 + lc_row;
        const bool horizon = (t + 1 >= K.nt);
        const int rx = K.gate_r ? __ldg(K.gate_r) : K.rx, ry = K.gate_r ? __ldg(K.gate_r + 1) : K.ry;

        // ---- per-row constants
        RowC R;
        R.ci = c % K.nx;
        R.cj = c / K.nx;
        R.x0 = R.y0 = R.ax = R.ay = R.base = R.base_hit = R.AB = 0.0;
        R.ilc = R.jlc = R.soff = 0;
        R.wi = R.wj = R.tslot = -1;
        R.rflags = 0;
        bool terminal = false;
        if (row_ok) {
            const int ci = R.ci, cj = R.cj;
            R.x0 = DADD(K.ox, DMUL(DADD((double)ci, 0.5), K.dx));   // environment.py:99-100
            R.y0 = DADD(K.oy, DMUL(DADD((double)cj, 0.5), K.dx));
            const fm_action A = K.act[a];
            R.ax = A.ax;
            R.ay = A.ay;
            R.base = A.base;
            R.base_hit = A.base_hit;
            terminal = (c == K.tcell);
            const bool obstacle = !terminal && K.mask[(size_t)t * K.nc + c];
            if (terminal || obstacle) R.rflags |= RF_DEAD;
            if (terminal) R.rflags |= RF_TERMINAL;
            if (!horizon) {
                // the reference's obstacle gate (model_builder.py:218-228, 339-345)
                if (box_count(K, t, ci - rx, ci + rx, cj - ry, cj + ry) > 0) {
                    R.rflags |= RF_GATE;
                    // an in-window segment only touches cells within one of the window
                    if (box_count(K, t, ci - K.hx - 1, ci + K.hx + 1, cj - K.hy - 1, cj + K.hy + 1) > 0)
                        R.rflags |= RF_SEGWIN;
                }
                if (box_count(K, t + 1, ci - K.hx, ci + K.hx, cj - K.hy, cj + K.hy) > 0) R.rflags |= RF_LANDWIN;
                if (K.obj == FM_OBJ_NET_ENERGY)
                    R.AB = DADD(A.neg_cff, DMUL(K.h_cr, K.g[(size_t)t * K.nc + c]));   // model_builder.py:358
            }
            // window [ci-hx, ci+hx] x [cj-hy, cj+hy] clipped to the grid: a
            // landing inside it is in-domain and inside the sub-grid
            R.ilc = max(ci - K.hx, 0);
            R.jlc = max(cj - K.hy, 0);
            R.wi = min(ci + K.hx, K.nx - 1) - R.ilc;
            R.wj = min(cj + K.hy, K.ny - 1) - R.jlc;
            R.soff = -((cj - K.hy) * W + (ci - K.hx));    // slot = j1*W + i1 + soff
            const int tci = K.tcell % K.nx, tcj = K.tcell / K.nx;
            if ((unsigned)(tci - R.ilc) <= (unsigned)R.wi && (unsigned)(tcj - R.jlc) <= (unsigned)R.wj)
                R.tslot = tcj * W + tci + R.soff;
        }
        // rows whose window is clipped by the domain boundary can land outside it
        const bool edge_row = row_ok && (R.ci - K.hx < 0 || R.ci + K.hx >= K.nx || R.cj - K.hy < 0 ||
                                         R.cj + K.hy >= K.ny);
        double S = 0.0;
        int viol = 0;
        // slots [s_lo, s_hi] (+ OUT) hold this row's nonzero counts: a lean
        // binned task narrows it to the slots its counts went to, so the
        // census and the fill below skip the window's empty slots
        int s_lo = 0, s_hi = nslot - 1;
        if (PART != 0) {
            const bool obst_task =
                !horizon && __any_sync(kFull, row_ok && (R.rflags & (RF_DEAD | RF_SEGWIN | RF_LANDWIN)));
            if (obst_task != OBST_PART) {   // the other launch's task
                // (bin-only launches get classified lists: a disagreement
                // would be a bug -- the list launch still builds the task)
                if (BINONLY && lane == 0) K.task_list[atomicAdd(K.task_list_n, 1u)] = task;
                continue;
            }
        }

        if (horizon) {
            // step_flat's horizon branch (model_builder.py:319-328): every
            // realization -> SINK with r_outbound, then the dead override.
            if (row_ok) {
                const double rw = terminal ? 0.0 : K.r_out;
                if (FLAGS & F_CNT) {
                    S = DADD(DMUL((double)nr, rw), 0.0);   // exact under F_CNT: the loop's sum
                } else {
                    for (int r = 0; r < nr; ++r) S = DADD(S, rw);
                }
                h16[nslot * 32] = (uint16_t)nr;
            }
        } else {
            const bool edge = __any_sync(kFull, edge_row);
            const unsigned rowmask = __ballot_sync(kFull, row_ok);   // lanes that run chunk_rows
            const bool obst = LEAN_PART   ? false
                              : OBST_PART ? true
                                          : __any_sync(kFull, row_ok && (R.rflags & (RF_DEAD | RF_SEGWIN | RF_LANDWIN)));
            const int DW = (nslot + 31) >> 5, CWD = 2 * DW;   // class words per cell
            if (obst) {
                // danger map: 2-bit class per (cell, window slot), 16 slots per
                // word: 0 safe, 1 landing cell masked at t+1, 2 gated with the
                // tight box [min(c,l), max(c,l)] touching the mask at t, 3
                // gated with only the box grown by one cell touching it
                for (int wd = 0; wd < CW * DW; ++wd) {
                    const int cs = wd / DW, sl = (wd - cs * DW) * 32 + lane;
                    const int lc = grp * CW + cs;
                    unsigned c = 0;
                    if (lc < K.ncell && sl < nslot) {
                        const int cc = K.cell0 + lc, cci = cc % K.nx, ccj = cc / K.nx;
                        const int li = cci + sl % W - K.hx, lj = ccj + sl / W - K.hy;
                        if ((unsigned)li < (unsigned)K.nx && (unsigned)lj < (unsigned)K.ny) {
                            if (K.mask[(size_t)(t + 1) * K.nc + lj * K.nx + li]) {
                                c = 1;
                            } else if (box_count(K, t, cci - rx, cci + rx, ccj - ry, ccj + ry) > 0 &&
                                       box_count(K, t, min(cci, li) - 1, max(cci, li) + 1, min(ccj, lj) - 1,
                                                 max(ccj, lj) + 1) > 0) {
                                // tight needs cell(x0) == source cell (host-checked)
                                c = (!K.src_cell_exact || box_count(K, t, min(cci, li), max(cci, li),
                                                                    min(ccj, lj), max(ccj, lj)) > 0) ? 2 : 3;
                                // ex == x1 exactly for this source: the tight box is the exact one
                                const bool ex_exact = (cci >= K.sx_lo || cci <= K.sx_hi) && (ccj >= K.sy_lo || ccj <= K.sy_hi);
                                if (c == 3 && ex_exact) c = 0;
                                // the landing cell itself masked at t: the last sample (frac = 1)
                                // is ex = x1 (Sterbenz), inside it -- every transition landing
                                // here is blocked (environment.py:359-367): settled as class 1
                                if (ex_exact && K.mask[(size_t)t * K.nc + lj * K.nx + li]) c = 1;
                            }
                        }
                    }
                    // pack: lane l's class -> bits 2(l & 15) of word (l >> 4)
                    const unsigned w0 = __ballot_sync(kFull, c & 1u), w1 = __ballot_sync(kFull, c & 2u);
                    if (lane < 2) {
                        unsigned lo = (w0 >> (16 * lane)) & 0xFFFFu, hi = (w1 >> (16 * lane)) & 0xFFFFu;
                        lo = (lo | (lo << 8)) & 0x00FF00FFu;   // spread 16 bits to even positions
                        lo = (lo | (lo << 4)) & 0x0F0F0F0Fu;
                        lo = (lo | (lo << 2)) & 0x33333333u;
                        lo = (lo | (lo << 1)) & 0x55555555u;
                        hi = (hi | (hi << 8)) & 0x00FF00FFu;
                        hi = (hi | (hi << 4)) & 0x0F0F0F0Fu;
                        hi = (hi | (hi << 2)) & 0x33333333u;
                        hi = (hi | (hi << 1)) & 0x55555555u;
                        danger[cs * CWD + (wd - cs * DW) * 2 + lane] = lo | (hi << 1);
                    }
                }
                __syncwarp();
            }
            const uint32_t *cls = danger + cs_row * CWD;
            // fast-path form of the row constants: target slot and OUT slot in
            // q = slot - soff coordinates, histogram pointer shifted by soff
            RowC Rf = R;
            Rf.tslot = R.tslot >= 0 ? R.tslot - R.soff : INT_MIN;
            const int outq = nslot - R.soff;
            uint16_t *h16q = h16 + R.soff * 32;
            bool binned = false;
            if constexpr (PART != 0 && (FLAGS & F_PROVEN) && (FLAGS & F_CNT)) {
                if (K.bin_ok) {
                    int q_lo = INT_MAX, q_hi = INT_MIN;   // q coordinates (slot - soff), OUT excluded
                    binned = bin_task<FLAGS, OBST_PART>(Kg, wbase, tab_s, t, grp, ag, Rf, outq, row_ok, cs_row,
                                                        half_one, danger, q_lo, q_hi);
                    if (LEAN_PART && binned) {
                        const bool any = q_lo <= q_hi;   // else every count is OUT
                        s_lo = any ? q_lo + R.soff : nslot;
                        s_hi = any ? q_hi + R.soff : nslot - 1;
                    }
#ifdef FM_STATS
                    tpath = binned ? 1 : 2;
#endif
                    if (BINONLY && !binned) {   // to the list launch (per-transition code)
                        if (lane == 0) K.task_list[atomicAdd(K.task_list_n, 1u)] = task;
                        // the bin regions overlay the per-transition histogram,
                        // which the next task (a horizon task) expects zeroed
                        uint4 *z = reinterpret_cast<uint4 *>(hist16);
                        for (int i = lane; i < (nslot + 1) * 4; i += 32) z[i] = make_uint4(0u, 0u, 0u, 0u);
                        __syncwarp();
                        continue;
                    }
                    if (binned) {
                        h16 = reinterpret_cast<uint16_t *>(wbase + K.off_bdense) + lane;
                    } else {
                        // the bin path's regions overlay this histogram: clear it
                        if (lane == 0) FM_STAT(7, 1);
                        for (int sl = 0; sl <= nslot; ++sl) h16[sl * 32] = 0;
                        __syncwarp();
                    }
                }
            }
            if (!BINONLY && !binned) {
            // stage the CW cells' modes
            for (int i = lane; i < CW * nm; i += 32) {
                const int cs = i / nm, m = i - (i / nm) * nm;
                const int lc = grp * CW + cs;
                if (lc < K.ncell)
                    modes_s[i] = *reinterpret_cast<const double2 *>(
                        K.modes + (((size_t)m * K.nt + t) * K.nc + K.cell0 + lc) * 2);
            }
            const int lc_rec = grp * CW + cs_rec;
            const bool rec_ok = rec_lane && lc_rec < K.ncell;
            double2 mu = make_double2(0.0, 0.0);
            if (rec_ok) mu = *reinterpret_cast<const double2 *>(K.mean + ((size_t)t * K.nc + K.cell0 + lc_rec) * 2);
            const double *cf_t = K.coeffs + (size_t)t * nr * nm;
            // even mode count and 16-byte aligned coefficient rows: pair layout
            const bool pairs = (nm & 1) == 0 && nm > 0 && ((reinterpret_cast<uintptr_t>(cf_t) & 15) == 0);
            const double *g_n = K.g + (size_t)(t + 1) * K.nc;
            // lean net-energy rows: table h_cr * g[t+1][landing cell] per
            // (cell, window slot), 0 outside the domain (model_builder.py:357-358)
            const double *hgq = g_n;
            if ((FLAGS & F_NET) && (FLAGS & F_PROVEN) && PART == 1) {
                double *hg = reinterpret_cast<double *>(wbase + K.off_hg);
                for (int i = lane; i < CW * nslot; i += 32) {
                    const int cs = i / nslot, sl = i - cs * nslot;
                    const int lc = grp * CW + cs;
                    double hv = 0.0;
                    if (lc < K.ncell) {
                        const int cc = K.cell0 + lc;
                        const int li = cc % K.nx + sl % W - K.hx, lj = cc / K.nx + sl / W - K.hy;
                        if ((unsigned)li < (unsigned)K.nx && (unsigned)lj < (unsigned)K.ny)
                            hv = DMUL(K.h_cr, g_n[lj * K.nx + li]);
                    }
                    hg[i] = hv;
                }
                hgq = hg + cs_row * nslot + R.soff;   // indexed by q = slot - soff
            }
            const double2 *vrow = vbuf + cs_row * (RC + 1);
            // chunk loader: coefficients [r0, r0+RC) x [0, nm) land transposed
            // as coefT[m][r - r0] (conflict-free reads in the reconstruction);
            // element-granular cp.async, contiguous (coalesced) global reads.
            auto issue_chunk = [&](int r0) {
                const int nrc = min(RC, nr - r0);
                const double *src = cf_t + (size_t)r0 * nm;
                if (pairs) {
                    // 16-byte copies: (realization rl, modes 2p..2p+1) -> coef2[p][rl]
                    // incremental (realization, pair) walk: no integer division
                    const int n_el = nrc * np2;
                    if (p_dp == 0) {
                        // np2 divides 32: this lane's pair is fixed and its
                        // realization advances by p_dr per step
                        const double *sp = src + p_r0 * nm + 2 * p_p0;
                        double *dp = coefT + (p_p0 * RC + p_r0) * 2;
                        for (int i = lane; i < n_el; i += 32, sp += p_dr * nm, dp += 2 * p_dr) cp_async16(dp, sp);
                        cp_async_commit();
                        return;
                    }
                    int rl = p_r0, pp = p_p0;
                    for (int i = lane; i < n_el; i += 32) {
                        cp_async16(coefT + (pp * RC + rl) * 2, src + rl * nm + 2 * pp);
                        rl += p_dr;
                        pp += p_dp;
                        if (pp >= np2) {
                            pp -= np2;
                            ++rl;
                        }
                    }
                } else {
                    const int n_el = nrc * nm;
                    src += lane;
                    int er = e_r0, em = e_m0;
                    for (int i = lane; i < n_el; i += 32, src += 32) {
                        cp_async8(coefT + em * RC + er, src);
                        er += e_dr;
                        em += e_dm;
                        if (em >= nm) {
                            em -= nm;
                            ++er;
                        }
                    }
                }
                cp_async_commit();
            };
            issue_chunk(0);
            for (int r0 = 0; r0 < nr; r0 += RC) {
                cp_async_wait_all();
                __syncwarp();
                if (rec_ok && pairs && nm == 8) {
                    recon_m8(modes_s + cs_rec * 8, reinterpret_cast<const double2 *>(coefT), mu, RC, RW, RPL, rr,
                             nr - r0, vbuf + cs_rec * (RC + 1));
                } else if (rec_ok) {
                    const double2 *md = modes_s + cs_rec * nm;
                    for (int p = 0; p < RPL; ++p) {
                        const int rl = p * RW + rr;
                        if (rl < RC && r0 + rl < nr) {
                            double vx = mu.x, vy = mu.y;
                            if (pairs) {
                                const double2 *c2 = reinterpret_cast<const double2 *>(coefT) + rl;
                                for (int m = 0; m < nm; m += 2) {   // environment.py:295-297, ascending m
                                    const double2 kk = c2[(m >> 1) * RC];
                                    const double2 ma = md[m], mb = md[m + 1];
                                    vx = DADD(vx, DMUL(kk.x, ma.x));
                                    vy = DADD(vy, DMUL(kk.x, ma.y));
                                    vx = DADD(vx, DMUL(kk.y, mb.x));
                                    vy = DADD(vy, DMUL(kk.y, mb.y));
                                }
                            } else {
                                for (int m = 0; m < nm; ++m) {   // environment.py:295-297, ascending m
                                    const double k = coefT[m * RC + rl];
                                    const double2 mm = md[m];
                                    vx = DADD(vx, DMUL(k, mm.x));
                                    vy = DADD(vy, DMUL(k, mm.y));
                                }
                            }
                            vbuf[cs_rec * (RC + 1) + rl] = make_double2(vx, vy);
                        }
                    }
                }
                __syncwarp();
                if (r0 + RC < nr) issue_chunk(r0 + RC);   // lands while the rows work
                const int nk = min(RC, nr - r0);
                if ((FLAGS & F_PROVEN) && (FLAGS & F_CNT) && obst) {
                    // whole warp (the drain is warp-cooperative); dead rows
                    // count nothing: no overflow test is needed under
                    // F_PROVEN and their counts are all OUT
                    chunk_rows_obst_cnt<FLAGS>(Kg, t, Rf, vrow, nk, cls, h16q, outq,
                                               row_ok && !(R.rflags & RF_DEAD), half_one, wbase + K.off_queue,
                                               (unsigned)__cvta_generic_to_shared(hist16), grp);
                } else if ((FLAGS & F_PROVEN) && obst) {
                    if (row_ok) chunk_rows_obst_seq<FLAGS>(Kg, t, Rf, vrow, nk, g_n, cls, h16q, outq, rowmask, S,
                                                           half_one);
                } else if (row_ok) {
                    FM_STAT(obst ? 3 : 4, nk);
                    if (obst) {
                        if (edge)
                            chunk_rows<FLAGS, true, true>(K, Kg, t, Rf, vrow, nk, g_n, cls, h16q, outq, rowmask, S,
                                                          viol);
                        else
                            chunk_rows<FLAGS, false, true>(K, Kg, t, Rf, vrow, nk, g_n, cls, h16q, outq, rowmask, S,
                                                           viol);
                    } else if (FLAGS & F_PROVEN) {
                        // F_CNT: edge rows count out-of-domain landings in their
                        // (unclipped) window slots and fold them into OUT below
#ifdef FM_NO_EDGE_FOLD
                        if (edge)
#else
                        if (edge && !(FLAGS & F_CNT))
#endif
                            chunk_rows_lean<FLAGS, true>(K, Rf, vrow, nk, hgq, h16q, outq, S, half_one);
                        else
                            chunk_rows_lean<FLAGS, false>(K, Rf, vrow, nk, hgq, h16q, outq, S, half_one);
                    } else {
                        if (edge)
                            chunk_rows<FLAGS, true, false>(K, Kg, t, Rf, vrow, nk, g_n, cls, h16q, outq, rowmask, S,
                                                           viol);
                        else
                            chunk_rows<FLAGS, false, false>(K, Kg, t, Rf, vrow, nk, g_n, cls, h16q, outq, rowmask,
                                                            S, viol);
                    }
                }
                asm volatile("" ::: "memory");   // histogram reductions (no clobber) before any plain access
                __syncwarp();
            }
            }   // !binned
            const bool dead_row = row_ok && (R.rflags & RF_DEAD);
            if ((FLAGS & F_CNT) && dead_row) h16[nslot * 32] = (uint16_t)nr;   // every realization -> SINK
            if ((FLAGS & F_CNT) && row_ok && edge_row && !dead_row) {
                // window slots whose cell lies outside the domain held the
                // landings that leave it: SINK (model_builder.py:331-335, 347)
                int extra = 0;
                for (int dj = -K.hy; dj <= K.hy; ++dj) {
                    const bool jout = (unsigned)(R.cj + dj) >= (unsigned)K.ny;
                    for (int di = -K.hx; di <= K.hx; ++di) {
                        if (jout || (unsigned)(R.ci + di) >= (unsigned)K.nx) {
                            uint16_t &cnt = h16[((dj + K.hy) * W + di + K.hx) * 32];
                            extra += cnt;
                            cnt = 0;
                        }
                    }
                }
                h16[nslot * 32] += (uint16_t)extra;
            }
            if ((FLAGS & F_CNT) && row_ok) {
                // exact reward sum from the counts (F_CNT): every partial sum
                // of the reference's sequential loop is exactly representable,
                // so it equals n_norm*base + n_hit*base_hit + n_out*r_out
                // (dead rows: all OUT; the target's rewards are 0.0);
                // + 0.0 turns a -0.0 into the loop's +0.0
                const int n_out = h16[nslot * 32], n_hit = R.tslot >= 0 ? h16[R.tslot * 32] : 0;
                if constexpr ((FLAGS & F_NET) != 0) {
                    // reward_mode 1 (counts): sum over landing slots, in slot
                    // order, of count x step_flat's net-energy reward
                    // ((-(c_f f f) + h_cr g_src + h_cr g_dst) dt, + r_term at
                    // the target; model_builder.py:357-360) -- agrees with the
                    // sequential sum to rounding.  Landings outside the domain
                    // were folded into OUT above.
                    S = 0.0;
                    if (!(R.rflags & RF_DEAD)) {
                        const double *g_n = K.g + (size_t)(t + 1) * K.nc;
                        // slots outside [s_lo, s_hi] hold no counts (a lean
                        // binned row's range, see the emission below)
                        for (int sl = s_lo; sl <= s_hi && sl < nslot; ++sl) {
                            const int cnt = h16[sl * 32];
                            if (!cnt) continue;
                            const int li = R.ci + sl % W - K.hx, lj = R.cj + sl / W - K.hy;
                            double b = DADD(R.AB, DMUL(K.h_cr, __ldg(g_n + lj * K.nx + li)));
                            if (!(FLAGS & F_DT_ONE)) b = DMUL(b, K.dt);
                            if (sl == R.tslot) b = DADD(b, K.r_term);
                            S = DADD(S, DMUL((double)cnt, b));
                        }
                    }
                    S = DADD(DADD(S, DMUL((double)n_out, K.r_out)), 0.0);
                } else {
                    const int n_norm = nr - n_out - n_hit;
                    S = DADD(DADD(DADD(DMUL((double)n_norm, R.base), DMUL((double)n_hit, R.base_hit)),
                                  DMUL((double)n_out, K.r_out)),
                             0.0);
                }
                if (R.rflags & RF_TERMINAL) S = 0.0;
            }
        }

        if (__any_sync(kFull, viol) && viol && row_ok) atomicOr(K.viol + (size_t)t * K.na + a, 1u);
#ifdef FM_STATS
        if (OBST_PART && lane == 0) {
            const unsigned slot = atomicAdd(&g_fm_tcount, 1u);
            const unsigned gw = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % (148 * 64);
            if (slot < (1u << 17)) {
                g_fm_ttimes[slot] = ((unsigned long long)task << 40) | ((unsigned long long)tpath << 36) |
                                    (unsigned long long)min(clock64() - tclk0, (long long)((1ll << 36) - 1));
                for (int k = 0; k < 8; ++k) {
                    g_fm_ttimes[(1u << 18) + slot * 8 + k] = g_fm_wcnt[gw][k];
                    g_fm_wcnt[gw][k] = 0;
                }
            }
        }
#endif

        // ---- emit: nnz census, warp scan, bump allocation, slot-ordered fill
        int nnz = 0;
        if (row_ok) {
            for (int sl = s_lo; sl <= s_hi; ++sl) nnz += h16[sl * 32] != 0;
            nnz += h16[nslot * 32] != 0;   // OUT
        }
        int incl = nnz;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(kFull, incl, 31);
        unsigned long long base_pos = 0;
        if (lane == 0) base_pos = atomicAdd(K.nnz_counter, (unsigned long long)total);
        base_pos = __shfl_sync(kFull, base_pos, 0);
        if (row_ok) {
            unsigned long long pos = base_pos + (unsigned long long)(incl - nnz);
            const size_t row = ((size_t)t * K.mncell + (c - K.mcell0)) * K.na + a;
            K.row_ptr[row] = pos;
            K.row_nnz[row] = (uint16_t)nnz;
            K.reward[row] = DDIV(S, (double)nr);   // finalize_rewards (model_builder.py:462-464)
            for (int sl = s_lo; sl <= nslot; ++sl) {
                if (sl == s_hi + 1) sl = nslot;   // past the range: the OUT slot
                const uint32_t x = h16[sl * 32];
                if (!x) continue;
                h16[sl * 32] = 0;
                if (pos < K.capacity) K.entries[pos] = ((uint32_t)sl << 16) | x;   // slots ascend = cols ascend
                ++pos;
            }
        }
        __syncwarp();
        if (PART != 0 && h16 != hist16 + lane) {
            // a binned task: its counters overlaid the per-transition
            // histogram, which every task expects zeroed
            uint4 *z = reinterpret_cast<uint4 *>(hist16);
            for (int i = lane; i < (nslot + 1) * 4; i += 32) z[i] = make_uint4(0u, 0u, 0u, 0u);
            __syncwarp();
        }
    }
}

// Recomputes one (t, a) sweep over every (r, c) of the layer to reproduce
// the reference's ContractViolation message (model_builder.py:430-438):
// argmax over non-sink entries of |di|+|dj|, first flat index r*N_c + c.
__global__ void k_viol_report(const __grid_constant__ BuildK K, int t, int a, int pass, unsigned long long *best,
                              int32_t *didj)
{
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)K.nr * K.nc) return;
    const int r = (int)(idx / K.nc), c = (int)(idx % K.nc);
    const int ci = c % K.nx, cj = c / K.nx;
    double vx = K.mean[((size_t)t * K.nc + c) * 2], vy = K.mean[((size_t)t * K.nc + c) * 2 + 1];
    for (int m = 0; m < K.nm; ++m) {
        const double k = K.coeffs[((size_t)t * K.nr + r) * K.nm + m];
        const double *md = K.modes + (((size_t)m * K.nt + t) * K.nc + c) * 2;
        vx = DADD(vx, DMUL(k, md[0]));
        vy = DADD(vy, DMUL(k, md[1]));
    }
    const fm_action A = K.act[a];
    const double x0 = DADD(K.ox, DMUL(DADD((double)ci, 0.5), K.dx));
    const double y0 = DADD(K.oy, DMUL(DADD((double)cj, 0.5), K.dx));
    const double x1 = DADD(x0, DMUL(DADD(vx, A.ax), K.dt)), y1 = DADD(y0, DMUL(DADD(vy, A.ay), K.dt));
    const int i1 = __double2int_rd(to_cell<0>(x1, K.ox, K.dx, K.inv_dx));
    const int j1 = __double2int_rd(to_cell<0>(y1, K.oy, K.dx, K.inv_dx));
    const bool inb = (unsigned)i1 < (unsigned)K.nx && (unsigned)j1 < (unsigned)K.ny;
    bool bad = !inb;
    if (inb) bad = K.mask[(size_t)(t + 1) * K.nc + j1 * K.nx + i1] != 0;
    const int rx = K.gate_r ? K.gate_r[0] : K.rx, ry = K.gate_r ? K.gate_r[1] : K.ry;
    if (!bad && box_count(K, t, ci - rx, ci + rx, cj - ry, cj + ry) > 0)
        bad = seg_blocked<0>(K, t, x0, y0, x1, y1);
    if (bad) return;
    const int di = i1 - ci, dj = j1 - cj;
    const unsigned long long key = (unsigned long long)(abs(di) + abs(dj));
    const unsigned long long packed = (key << 40) | (0xFFFFFFFFFFull - (unsigned long long)idx);
    if (pass == 0) {
        atomicMax(best, packed);
    } else if (packed == *best) {
        didj[0] = di;
        didj[1] = dj;
    }
}

static int align16(int x) { return (x + 15) & ~15; }

static int smem_block_optin()
{
    static int v = 0;
    if (!v) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || v <= 0)
            v = 232448;
        cudaGetLastError();
    }
    return v;
}

// Per-warp shared memory: u16 histogram [nslot+1][32] | v chunk [CW][RC+1]
// | transposed coefficients [nm][RC] | modes [CW][nm] | danger classes
// [CW][2 words per 32 slots] | (queue entries) deferred exact tests.
static void smem_layout(BuildK &K, int RC, int queue, bool hg = false, bool ghist = false)
{
    K.RC = RC;
    K.off_vbuf = ghist ? 0 : align16((K.nslot + 1) * 64);
    K.off_coef = K.off_vbuf + K.CW * (K.RC + 1) * (int)sizeof(double2);
    K.off_modes = align16(K.off_coef + K.RC * K.nm * (int)sizeof(double));
    K.off_danger = align16(K.off_modes + K.CW * K.nm * (int)sizeof(double2));
    K.off_queue = align16(K.off_danger + 2 * K.CW * ((K.nslot + 31) / 32) * 4);
    K.off_hg = align16(K.off_queue + queue * (int)sizeof(QItem));
    K.smem_warp = align16(K.off_hg + (hg ? K.CW * K.nslot * (int)sizeof(double) : 0));
}

// Largest chunk (64 or 32 realizations, >= RW) whose per-warp layout still
// fits 4 blocks of 4 warps per SM; the smallest if none does.
static void smem_layout_fit(BuildK &K, int queue, bool hg)
{
    static int smem_sm = 0;
    if (!smem_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess ||
            smem_sm <= 0)
            smem_sm = 233472;
        cudaGetLastError();
    }
    // resident warps per SM with 4-warp blocks (capped at 16); more warps
    // win, the larger chunk on a tie (wide sub-grids: neither fits 16 warps
    // and the 64-realization chunk measured faster, 98.9 vs 111.0 ms)
    const int cands[2] = {K.RW >= FM_BUILD_RC ? K.RW : FM_BUILD_RC, K.RW >= 32 ? K.RW : 32};
    int best = 0, best_w = -1;
    for (int i = 0; i < 2; ++i) {
        smem_layout(K, cands[i], queue, hg);
        int blocks = smem_sm / (4 * K.smem_warp + 1024);
        if (blocks > 4) blocks = 4;
        if (4 * blocks > best_w) {
            best_w = 4 * blocks;
            best = i;
        }
    }
    smem_layout(K, cands[best], queue, hg);
}

// Per-warp regions of the bin path, overlaid on the legacy layout after the
// dense histogram: bin counters | coefficient ring | deferred queue.  The
// counters take whatever the legacy layout leaves (at least 512 words), so
// the bin path costs no occupancy when it fits.
static void bin_layout(BuildK &K)
{
    const int ring = kBinRing * 32 * 32, dense = (K.nslot + 1) * 64, q = kBinQ * 4;
    const int uni = align16(ring > dense ? ring : dense);
    K.off_bins = 0;
    int words = ((K.smem_warp - uni - q) / 4) & ~31;
    const char *ev = getenv("FM_BIN_WORDS");   // dev override (A/B of the occupancy trade-off)
    const int floor_words = ev ? atoi(ev) : (K.CW >= 2 ? FM_BIN_WORDS2 : 2048);
    if (words < floor_words) words = floor_words;
    K.bin_words = words;
    K.off_bdense = align16(words * 4);
    K.off_bring = K.off_bdense;
    K.off_bq = K.off_bdense + uni;
    const int end = align16(K.off_bq + q);
    if (end > K.smem_warp) K.smem_warp = end;
    K.off_block = align16(2 * (K.bin_ns + 1) * kBinRep * (int)sizeof(BinEnt));
}

// Lean tasks in a bin-only launch (PART 3): bin counters | ring, later the
// dense histogram | queue, nothing of the per-transition layout but its
// histogram (horizon tasks), so more warps fit per SM.
static void bin_layout_lean(BuildK &K)
{
    const int ring = kBinRing * 32 * 32, dense = (K.nslot + 1) * 64, q = kBinQ * 4;
    const int uni = align16(ring > dense ? ring : dense);
    const int words = K.CW >= 2 ? FM_BIN_WORDS2 : 2048;
    K.bin_words = words;
    K.off_bins = 0;
    K.off_bdense = align16(words * 4);
    K.off_bring = K.off_bdense;
    K.off_bq = K.off_bdense + uni;
    const int end = align16(K.off_bq + q);
    K.smem_warp = end > align16(dense) ? end : align16(dense);
    K.off_block = align16(2 * (K.bin_ns + 1) * kBinRep * (int)sizeof(BinEnt));
}

// Obstacle tasks (PART 2) by binning: bin counters | coefficient ring
// (kBinRingO chunks) | dense histogram | queue (kBinQO), all live at once
// (the queue drains mid-loop), then the danger map past both this and the
// per-transition layout (a task that cannot bin falls back to the latter).
// False when it does not fit a block's shared memory.
static bool bin_layout_obst(BuildK &K)
{
    const int legacy_end = K.smem_warp;
    const int words = K.CW >= 2 ? 1024 : 2048;
    K.bin_words = words;
    K.off_bins = 0;
    K.off_bring = align16(words * 4);
    K.off_bdense = align16(K.off_bring + kBinRingO * 32 * 32);
    K.off_bq = align16(K.off_bdense + (K.nslot + 1) * 64);
    const int end = align16(K.off_bq + kBinQO * 4 + (int)sizeof(ObstDrainBuf) +
                            K.CW * (2 * K.hx + 3) * (2 * K.hy + 3));
    K.off_danger = align16(end > legacy_end ? end : legacy_end);
    K.smem_warp = align16(K.off_danger + 2 * K.CW * ((K.nslot + 31) / 32) * 4);
    // bin tables, then fl(q / n) for n <= kFracSmemN
    K.off_block = align16(2 * (K.bin_ns + 1) * kBinRep * (int)sizeof(BinEnt) +
                          (kFracSmemN + 1) * (kFracSmemN + 2) / 2 * (int)sizeof(double));
    return K.off_block + K.smem_warp <= smem_block_optin();
}

// warp-aggregated append of val to list (when pred)
__device__ __forceinline__ void list_append(unsigned int *list, unsigned int *n, bool pred, unsigned int val)
{
    const unsigned act = __activemask(), m = __ballot_sync(act, pred);
    if (!m) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(n, (unsigned)__popc(m));
    base = __shfl_sync(act, base, leader);
    if (pred) list[base + __popc(m & ((1u << lane) - 1u))] = val;
}

// Task classes for the bin-only launches, with k_build's own test (a task is
// an obstacle task when a row of it is dead or has the mask near its window,
// model_builder.py:218-228, 247-259, 336-345): lean tasks (and the horizon)
// -> list 0; obstacle tasks with the mask within two cells of a source cell
// at t or t+1 (the slow ones: many exact transit tests) -> list 1; the
// other obstacle tasks -> list 2.  lists = 3 arrays of n_tasks, n = 3 counters.
__global__ void k_classify(const __grid_constant__ BuildK K, unsigned int *lists, unsigned int *n)
{
    const long long task = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (task >= K.n_tasks) return;
    const int per_t = K.groups * K.nag;
    const int t = K.t0 + (int)(task / per_t);
    const int grp = (int)(task % per_t) / K.nag;
    const int rx = K.gate_r ? __ldg(K.gate_r) : K.rx, ry = K.gate_r ? __ldg(K.gate_r + 1) : K.ry;
    bool obst = false, near = false;
    if (t + 1 < K.nt) {
        for (int cs = 0; cs < K.CW; ++cs) {
            const int lc = grp * K.CW + cs;
            if (lc >= K.ncell) break;
            const int c = K.cell0 + lc, ci = c % K.nx, cj = c / K.nx;
            const bool dead = c == K.tcell || K.mask[(size_t)t * K.nc + c];
            const bool segwin = box_count(K, t, ci - rx, ci + rx, cj - ry, cj + ry) > 0 &&
                                box_count(K, t, ci - K.hx - 1, ci + K.hx + 1, cj - K.hy - 1, cj + K.hy + 1) > 0;
            const bool landwin = box_count(K, t + 1, ci - K.hx, ci + K.hx, cj - K.hy, cj + K.hy) > 0;
            obst |= dead || segwin || landwin;
            near |= box_count(K, t, ci - 2, ci + 2, cj - 2, cj + 2) > 0 ||
                    box_count(K, t + 1, ci - 2, ci + 2, cj - 2, cj + 2) > 0;
        }
    }
    const int cls = !obst ? 0 : near ? 1 : 2;
    for (int k = 0; k < 3; ++k) list_append(lists + (size_t)k * K.n_tasks, n + k, cls == k, (unsigned)task);
}

template <int FL, int PART>
static int32_t launch_build_p(const BuildK &K, size_t smem, cudaStream_t s)
{
    (void)smem;   // recomputed: 4 warps per block, fewer when a warp's layout is large
    auto kern = k_build<FL, PART>;
    static int max_block = 0;
    if (!max_block) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&max_block, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
            max_block <= 0)
            max_block = 232448;
        cudaGetLastError();
    }
    int wpb = (max_block - K.off_block) / K.smem_warp;
    if (wpb > 4) wpb = 4;
    if (wpb < 1)
        return fm_fail(FM_BAD_ARG,
                       "sub-grid of %d slots needs %d B of shared memory per warp (at most %d per block on this "
                       "device)",
                       K.nslot + 1, K.smem_warp, max_block);
    const size_t bytes = (size_t)K.off_block + (size_t)wpb * K.smem_warp;
    FM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    int occ = 0;
    FM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * wpb, bytes));
    if (occ < 1) return fm_fail(FM_BAD_ARG, "k_build: %zu B smem per block does not fit", bytes);
    FM_CK(cudaMemsetAsync(K.task_counter, 0, sizeof(unsigned int), s));
    int sms = sm_count() - K.reserve_sms;
    if (sms < 1) sms = 1;
    // the list launch (tasks the bin-only launches could not bin: usually
    // none or a few dozen) runs on a small grid -- most of its cost is launch
    const int blocks = (PART == 0 && K.task_list) ? (sms + 3) / 4 : occ * sms;
    kern<<<blocks, 32 * wpb, bytes, s>>>(K);
    FM_CK_LAUNCH("k_build");
    return FM_OK;
}

template <int FL>
static int32_t launch_build_t(const BuildK &K, size_t smem, cudaStream_t s, int phases)
{
    if constexpr (!(FL & F_PROVEN)) {
        return (phases & 1) ? launch_build_p<FL, 0>(K, smem, s) : FM_OK;   // one class: the lean phase
    } else {
        int32_t st = FM_OK;
        if constexpr ((FL & F_CNT) != 0) {
            if (K.bin_ok && !getenv("FM_NO_BINONLY")) {
                // bin-only launches (lean, then obstacle tasks); the tasks
                // they cannot bin run per transition in a PART 0 launch over
                // the list they append to
                // lists: [lean | near-obstacle | other obstacle | failed] x n_tasks, then 4 counters
                unsigned int *list = nullptr;
                const size_t nt4 = 4 * (size_t)K.n_tasks;
                FM_CK(cudaMallocAsync(reinterpret_cast<void **>(&list), sizeof(unsigned int) * (nt4 + 4), s));
                FM_CK(cudaMemsetAsync(list + nt4, 0, 4 * sizeof(unsigned int), s));
                unsigned int *cnt = list + nt4;
                k_classify<<<(unsigned)((K.n_tasks + 255) / 256), 256, 0, s>>>(K, list, cnt);
                FM_CK_LAUNCH("k_classify");
                BuildK K1 = K;
                K1.task_list = list + 3 * (size_t)K.n_tasks;
                K1.task_list_n = cnt + 3;
                K1.src_a = list;
                K1.src_a_n = cnt;
                K1.src_b = nullptr;
                K1.src_b_n = cnt + 3;   // unused with src_b null
                if (phases & 1) {
                    BuildK K3 = K1;
                    bin_layout_lean(K3);
                    st = launch_build_p<FL, 3>(K3, (size_t)4 * K3.smem_warp, s);
                }
                if (st == FM_OK && (phases & 2)) {
                    BuildK K2 = K1;
                    K2.src_a = list + (size_t)K.n_tasks;
                    K2.src_a_n = cnt + 1;
                    K2.src_b = list + 2 * (size_t)K.n_tasks;
                    K2.src_b_n = cnt + 2;
                    K2.off_block = 0;
                    smem_layout_fit(K2, kQueue, false);
                    if (!getenv("FM_NO_OBST_BINS") && bin_layout_obst(K2)) {
                        st = launch_build_p<FL, 4>(K2, (size_t)4 * K2.smem_warp, s);
                    } else {
                        K2.bin_ok = 0;
                        K2.off_block = 0;
                        smem_layout_fit(K2, kQueue, false);
                        st = launch_build_p<FL, 2>(K2, (size_t)4 * K2.smem_warp, s);
                    }
                }
                if (st == FM_OK) {
                    BuildK K0 = K1;
                    K0.bin_ok = 0;
                    K0.off_block = 0;
                    smem_layout_fit(K0, kQueue, false);
                    st = launch_build_p<FL, 0>(K0, (size_t)4 * K0.smem_warp, s);
                }
                FM_CK(cudaFreeAsync(list, s));
                return st;
            }
        }
        if (phases & 1) {
            if constexpr ((FL & F_NET) != 0) {
                // lean net-energy rows read h_cr * g[t+1] from a per-warp slot
                // table (half-size chunks keep 4 blocks per SM)
                BuildK K1 = K;
                K1.off_block = 0;
                smem_layout_fit(K1, 0, true);
                st = launch_build_p<FL, 1>(K1, (size_t)4 * K1.smem_warp, s);
            } else {
                st = launch_build_p<FL, 1>(K, smem, s);
            }
        }
        if (st != FM_OK || !(phases & 2)) return st;
        if constexpr ((FL & F_CNT) != 0) {
            // obstacle part: per-warp queue of deferred exact segment tests
            // (half-size reconstruction chunks keep it at 4 blocks per SM)
            BuildK K2 = K;
            K2.off_block = 0;
            smem_layout_fit(K2, kQueue, false);
            if (K2.bin_ok && (getenv("FM_NO_OBST_BINS") || !bin_layout_obst(K2))) {
                K2.bin_ok = 0;
                K2.off_block = 0;
                smem_layout_fit(K2, kQueue, false);
            }
            return launch_build_p<FL, 2>(K2, (size_t)4 * K2.smem_warp, s);
        } else {
            BuildK K2 = K;
            K2.off_block = 0;
            return launch_build_p<FL, 2>(K2, smem, s);
        }
    }
}

// Sub-grids whose histogram exceeds a block's shared memory: the checked
// kernel with the histogram in a stream-ordered global scratch buffer, one
// slice per warp of a persistent grid (tasks come from the task counter, so
// any grid size covers them; the grid shrinks to keep the scratch <= 4 GiB).
template <int FL>
static int32_t launch_build_ghist(BuildK K, cudaStream_t s)
{
    auto kern = k_build<FL, 0>;
    int max_block = 0, dev = 0;
    FM_CK(cudaGetDevice(&dev));
    FM_CK(cudaDeviceGetAttribute(&max_block, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    int wpb = max_block / K.smem_warp;
    if (wpb > 4) wpb = 4;
    if (wpb < 1)
        return fm_fail(FM_BAD_ARG, "sub-grid of %d slots: %d B of per-warp state exceed a block's shared memory",
                       K.nslot + 1, K.smem_warp);
    const size_t bytes = (size_t)wpb * K.smem_warp;
    FM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    int occ = 0;
    FM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * wpb, bytes));
    if (occ < 1) return fm_fail(FM_BAD_ARG, "k_build: %zu B smem per block does not fit", bytes);
    const size_t per_block = (size_t)wpb * (size_t)(K.nslot + 1) * 64;
    long long blocks = (long long)occ * sm_count();
    const long long cap = (long long)((4ull << 30) / per_block);
    if (blocks > cap) blocks = cap > 0 ? cap : 1;
    FM_CK(cudaMallocAsync(reinterpret_cast<void **>(&K.ghist), (size_t)blocks * per_block, s));
    FM_CK(cudaMemsetAsync(K.task_counter, 0, sizeof(unsigned int), s));
    kern<<<(unsigned)blocks, 32 * wpb, bytes, s>>>(K);
    FM_CK_LAUNCH("k_build");
    FM_CK(cudaFreeAsync(K.ghist, s));
    return FM_OK;
}

static int32_t launch_build(const BuildK &K, int flags, size_t smem, cudaStream_t s, int phases)
{
    if (flags & F_GHIST) {
        if (!(phases & 1)) return FM_OK;   // one class: the lean phase
        // identity geometry flags dropped: x*1, x/1, x-0 are exact
        if (flags & F_NET) return launch_build_ghist<F_GHIST | F_NET>(K, s);
        return launch_build_ghist<F_GHIST>(K, s);
    }
    if (flags & F_PROVEN) {
        // lean variants exist for the identity geometry (dt = dx = 1, origin
        // 0) and the general one; dropping identity flags never changes a
        // result (x*1, x/1, x-0 are exact)
        const int geo = (flags & 15) == (F_DT_ONE | F_OX_ZERO | F_DX_ONE) ? (flags & 15) : 0;
        switch (geo | (flags & (F_NET | F_PROVEN | F_CNT))) {
#define FM_CASE(F) \
    case F: return launch_build_t<F>(K, smem, s, phases);
            FM_CASE(11 | F_PROVEN) FM_CASE(11 | F_PROVEN | F_CNT) FM_CASE(11 | F_PROVEN | F_NET)
            FM_CASE(11 | F_PROVEN | F_CNT | F_NET)
            FM_CASE(F_PROVEN) FM_CASE(F_PROVEN | F_CNT) FM_CASE(F_PROVEN | F_NET) FM_CASE(F_PROVEN | F_CNT | F_NET)
#undef FM_CASE
        }
        return fm_fail(FM_BAD_ARG, "k_build: bad flags %d", flags);
    }
    switch (flags) {
#define FM_CASE(F) \
    case F: return launch_build_t<F>(K, smem, s, phases);
        FM_CASE(0) FM_CASE(1) FM_CASE(2) FM_CASE(3) FM_CASE(4) FM_CASE(5) FM_CASE(6) FM_CASE(7)
        FM_CASE(8) FM_CASE(9) FM_CASE(10) FM_CASE(11) FM_CASE(16) FM_CASE(17) FM_CASE(18) FM_CASE(19)
        FM_CASE(20) FM_CASE(21) FM_CASE(22) FM_CASE(23) FM_CASE(24) FM_CASE(25) FM_CASE(26) FM_CASE(27)
#undef FM_CASE
    }
    return fm_fail(FM_BAD_ARG, "k_build: bad flags %d", flags);
}

static bool is_pow2(double x)
{
    if (!(x > 0.0)) return false;
    int e;
    double m = frexp(x, &e);
    return m == 0.5;
}


// One axis of the lean-path proof.  reach = fl(fl(vmax + amax) * dt) bounds
// |fl(fl(v + a) * dt)| for every transition (|v| <= vmax exactly: it is the
// maximum of these very reconstructions; rounding is monotone), so
// x1 = fl(x0 + p) lies in [fl(x0 - reach), fl(x0 + reach)] and, by
// monotonicity of (x - o) / dx and floor, the landing index lies between the
// floors of the two ends.  Checked for every source index of the axis.
static bool prove_axis(int n, double o, double dx, double reach, int hw)
{
    for (int c = 0; c < n; ++c) {
        const double x0 = o + ((double)c + 0.5) * dx;   // environment.py:99-100
        const double ulo = ((x0 - reach) - o) / dx, uhi = ((x0 + reach) - o) / dx;
        if (!(fabs(ulo) < 0x1p30 && fabs(uhi) < 0x1p30)) return false;
        if (floor(ulo) - c < -hw || floor(uhi) - c > hw) return false;
    }
    return true;
}

// Every cell centre x0 = o + (c + 0.5) dx maps back to its own cell under
// the reference's (x - o) / dx and floor (environment.py:99-100, 358-362).
static bool source_cells_exact(const fm_grid &G)
{
    for (int c = 0; c < (G.nx > G.ny ? G.nx : G.ny); ++c) {
        if (c < G.nx && floor(((G.ox + ((double)c + 0.5) * G.dx) - G.ox) / G.dx) != c) return false;
        if (c < G.ny && floor(((G.oy + ((double)c + 0.5) * G.dx) - G.oy) / G.dx) != c) return false;
    }
    return true;
}

// Sterbenz ranges of one axis: with x1 in [fl(x0 - R), fl(x0 + R)] and
// x1 / 2 <= x0 <= 2 x1 (same sign), x1 - x0 is exact, so x0 + (x1 - x0)
// rounds to x1 itself.  lo = first index from which every larger index
// qualifies (positive side), hi = last index up to which every smaller one
// qualifies (negative side).
static void sterbenz_axis(int n, double o, double dx, double R, int &lo, int &hi)
{
    auto ok = [&](int c) {
        const double x0 = o + ((double)c + 0.5) * dx, a = x0 - R, b = x0 + R;
        if (a > 0.0) return x0 <= 2.0 * a && b <= 2.0 * x0;
        if (b < 0.0) return -x0 <= -2.0 * b && -a <= -2.0 * x0;
        return false;
    };
    lo = n;
    while (lo > 0 && ok(lo - 1)) --lo;
    hi = -1;
    while (hi + 1 < n && ok(hi + 1)) ++hi;
}

static bool prove_lean(const fm_build_args *h)
{
    const double vx = h->vmax_x, vy = h->vmax_y;
    if (!(vx >= 0.0 && vy >= 0.0 && std::isfinite(vx) && std::isfinite(vy))) return false;
    double ax = 0.0, ay = 0.0;
    for (int a = 0; a < h->n_actions; ++a) {
        const double x = fabs(h->h_actions[a].ax), y = fabs(h->h_actions[a].ay);
        if (!(x <= DBL_MAX && y <= DBL_MAX)) return false;
        ax = x > ax ? x : ax;
        ay = y > ay ? y : ay;
    }
    const fm_grid &G = h->grid;
    const double rx = (vx + ax) * G.dt, ry = (vy + ay) * G.dt;
    return std::isfinite(rx) && std::isfinite(ry) && prove_axis(G.nx, G.ox, G.dx, rx, h->hx) &&
           prove_axis(G.ny, G.oy, G.dx, ry, h->hy);
}

// Smallest k >= 0 with v * 2^k an integer (v finite), or -1.
static int dyadic_scale(double v)
{
    if (v == 0.0) return 0;
    if (!std::isfinite(v)) return -1;
    int e;
    const double f = frexp(fabs(v), &e);               // v = f 2^e, f in [0.5, 1)
    uint64_t m = (uint64_t)ldexp(f, 53);               // exact 53-bit mantissa
    const int tz = __builtin_ctzll(m);
    const int k = 53 - e - tz;
    return k > 0 ? k : 0;
}

// F_CNT precondition: every per-transition reward value (base, base_hit per
// action, r_outbound, 0) is an integer multiple of 2^-K and
// n_real * max|value| * 2^K <= 2^52, so every partial sum of the
// reference's sequential loop, and each count * value, is exact.
static bool rewards_sum_exactly(const fm_build_args *h)
{
    std::vector<double> vals{h->reward.r_outbound, 0.0};
    for (int a = 0; a < h->n_actions; ++a) {
        vals.push_back(h->h_actions[a].base);
        vals.push_back(h->h_actions[a].base_hit);
    }
    int K = 0;
    double mx = 0.0;
    for (double v : vals) {
        const int k = dyadic_scale(v);
        if (k < 0 || k > 900) return false;
        K = k > K ? k : K;
        mx = fabs(v) > mx ? fabs(v) : mx;
    }
    return ldexp(mx, K) * (double)h->env.n_real <= 0x1p52;
}

// Bin structure of one axis (see kBinNS): per action gamma / cluster index,
// clusters of step positions theta_a in (0, 1) and the bucket table.  Steps
// closer than 2 dzone + a bucket (plus margin) apart share one cluster, whose
// zone [min - dzone, max + dzone] routes realizations to the exact path, so
// every realization outside all zones lies on one side of every step of the
// cluster; steps near 0 or 1 join the unit boundary (always / never).
static bool bin_axis(const std::vector<double> &comp, double p, double dz, int NS, int &k1, BinEnt *tab, int *g,
                     int *r)
{
    const double eta = 1.0 / (8.0 * NS), gap = 1.0 / NS + 2.0 * eta;
    double hi0 = dz, lotop = 1.0 - dz;
    std::vector<int> bottom, top;
    std::vector<std::pair<double, int>> th;
    for (size_t a = 0; a < comp.size(); ++a) {
        const double c = 0.5 + comp[a] / p;
        if (!std::isfinite(c) || fabs(c) > 0x1p20) return false;
        const double gam = floor(c), beta = c - gam;
        g[a] = (int)gam;
        const double theta = beta > 0.0 ? 1.0 - beta : 1.0;
        if (theta <= 2.0 * dz + gap) {
            bottom.push_back((int)a);
            hi0 = fmax(hi0, theta + dz);
        } else if (theta >= 1.0 - 2.0 * dz - gap) {
            top.push_back((int)a);
            lotop = fmin(lotop, theta - dz);
        } else {
            th.push_back({theta, (int)a});
        }
    }
    std::sort(th.begin(), th.end());
    std::vector<double> clo, chi;
    std::vector<std::vector<int>> mem;
    for (auto &e : th) {
        if (!clo.empty() && e.first - dz - chi.back() <= gap) {
            chi.back() = e.first + dz;
            mem.back().push_back(e.second);
        } else {
            clo.push_back(e.first - dz);
            chi.push_back(e.first + dz);
            mem.push_back({e.second});
        }
    }
    while (!clo.empty() && clo.front() - hi0 <= gap) {
        hi0 = fmax(hi0, chi.front());
        bottom.insert(bottom.end(), mem.front().begin(), mem.front().end());
        clo.erase(clo.begin()); chi.erase(chi.begin()); mem.erase(mem.begin());
    }
    while (!clo.empty() && lotop - chi.back() <= gap) {
        lotop = fmin(lotop, clo.back());
        top.insert(top.end(), mem.back().begin(), mem.back().end());
        clo.pop_back(); chi.pop_back(); mem.pop_back();
    }
    if (!(hi0 + gap < lotop)) return false;
    const int K = (int)clo.size();
    k1 = K + 1;
    for (int a : bottom) r[a] = 0;
    for (int a : top) r[a] = K + 1;
    for (int k = 0; k < K; ++k)
        for (int a : mem[k]) r[a] = k + 1;
    if (K + 2 > 63) return false;   // kb + 1 must fit the 6 packed bits
    auto rd = [](double x) { return std::nextafter((float)x, -INFINITY); };
    auto ru = [](double x) { return std::nextafter((float)x, INFINITY); };
    // lo rounded down past its low 6 mantissa bits, which then carry kb + 1
    auto pack = [](float lo, int kb) {
        int b;
        memcpy(&b, &lo, 4);
        b = lo >= 0.0f ? ((b - 64) & ~63) : ((b + 64) & ~63);   // smaller value either way
        b |= kb + 1;
        float r;
        memcpy(&r, &b, 4);
        return r;
    };
    for (int b = 0; b <= NS; ++b) {   // entry NS: frac == 1
        const double elo = (double)b / NS - eta, ehi = (double)(b + 1) / NS + eta;
        int kb = 0;
        for (int k = 0; k < K; ++k) kb += chi[k] < elo ? 1 : 0;
        float lo = 3.0f, hi = 3.0f;
        int hits = 0;
        if (hi0 >= elo) { kb = -1; lo = -1.0f; hi = ru(hi0); ++hits; }
        for (int k = 0; k < K; ++k)
            if (clo[k] <= ehi && chi[k] >= elo) { kb = k; lo = rd(clo[k]); hi = ru(chi[k]); ++hits; }
        if (lotop <= ehi) { kb = K; lo = rd(lotop); hi = 2.0f; ++hits; }
        if (hits > 1) return false;
        tab[b] = BinEnt{pack(lo, kb), hi};
    }
    return true;
}

// Enables the bin path for a proven, count-formed build: tables, error
// allowances, per-action parameters.  dzone is sized for a reconstruction
// magnitude T of 3 vmax + 1; cells with a larger bound take the
// per-transition path (bin_setup).
static void bin_params(const fm_build_args *h, BuildK &K)
{
    K.bin_ok = 0;
    const fm_grid &G = h->grid;
    // at most two cells per task: the dense histogram overlays the
    // coefficient ring, so a task's cells are binned in one pass
    if (K.nm > 8 || K.na > kBinMaxA || K.CW > 2 || !h->h_actions) return;
    const double p = G.dx / G.dt;
    if (!(p > 0.0) || !std::isfinite(p)) return;
    const double vmax = fmax(h->vmax_x, h->vmax_y);
    double amax = 0.0;
    std::vector<double> ax(K.na), ay(K.na);
    for (int a = 0; a < K.na; ++a) {
        ax[a] = h->h_actions[a].ax;
        ay[a] = h->h_actions[a].ay;
        amax = fmax(amax, fmax(fabs(ax[a]), fabs(ay[a])));
    }
    // the reference's own roundings in the landing index (cell units): a
    // handful of roundings of magnitudes below M / dx
    const double M = fmax(fmax(fabs(G.ox), fabs(G.ox + G.nx * G.dx)), fmax(fabs(G.oy), fabs(G.oy + G.ny * G.dx))) +
                     (vmax + amax) * G.dt + G.dx;
    K.bin_eps = 0x1p-48 * (M / G.dx + 2.0);
    const double T = 3.0 * vmax + 1.0, ip = 1.0 / p;
    const double kRel = (2.0 * K.nm + 8.0) * 0x1p-24 * 1.001;
    K.bin_dzone = fmax(0x1p-17, 2.0 * (T * kRel * ip + 0x1p-21 * (T * ip + 1.0) + K.bin_eps));
    std::vector<int> gx(K.na), rx(K.na), gy(K.na), ry(K.na);
    if (!bin_axis(ax, p, K.bin_dzone, kBinNS, K.bin_k1x, K.tab, gx.data(), rx.data())) return;
    if (!bin_axis(ay, p, K.bin_dzone, kBinNS, K.bin_k1y, K.tab + kBinNS + 1, gy.data(), ry.data())) return;
    K.bin_ns = kBinNS;
    // coarser buckets shrink the replicated block-shared tables; accepted
    // only when they give the same step clusters (hence the same zones)
    for (int ns : {32, 64}) {
        BinEnt tab[2 * (kBinNS + 1)];
        int k1x = 0, k1y = 0;
        if (bin_axis(ax, p, K.bin_dzone, ns, k1x, tab, gx.data(), rx.data()) &&
            bin_axis(ay, p, K.bin_dzone, ns, k1y, tab + kBinNS + 1, gy.data(), ry.data()) && k1x == K.bin_k1x &&
            k1y == K.bin_k1y) {
            memcpy(K.tab, tab, sizeof(tab));
            K.bin_ns = ns;
            break;
        }
        bin_axis(ax, p, K.bin_dzone, kBinNS, k1x, K.tab, gx.data(), rx.data());   // restore
        bin_axis(ay, p, K.bin_dzone, kBinNS, k1y, K.tab + kBinNS + 1, gy.data(), ry.data());
    }
    for (int a = 0; a < K.na; ++a) K.bact[a] = BinAct{gx[a], rx[a], gy[a], ry[a]};
    K.bin_p = p;
    K.bin_p1 = p == 1.0 ? 1 : 0;
    K.bin_ip = (float)ip;
    K.envelope = reinterpret_cast<const int4 *>(h->envelope);
    K.bin_ok = 1;
    bin_layout(K);
    if (getenv("FM_BIN_DEBUG"))
        fprintf(stderr, "bin: ns %d k1 (%d, %d) dzone %.3g words %d smem_warp %d off_block %d\n", K.bin_ns, K.bin_k1x,
                K.bin_k1y, K.bin_dzone, K.bin_words, K.smem_warp, K.off_block);
}

// validates the arguments and fills the kernel parameter block + flags
static int32_t build_params(const fm_build_args *h, const fm_model *M, BuildK &K, int &flags)
{
    const fm_grid &G = h->grid;
    if (G.nx < 1 || G.ny < 1 || G.nt < 1 || !(G.dx > 0) || !(G.dt > 0))
        return fm_fail(FM_BAD_ARG, "fm_build: bad grid");
    if (h->env.n_modes < 0 || h->env.n_modes > 512) return fm_fail(FM_BAD_ARG, "fm_build: n_modes must be in [0,512]");
    if (h->env.n_real < 1 || h->env.n_real > 65535) return fm_fail(FM_BAD_ARG, "fm_build: n_real must be in [1,65535]");
    if (h->n_actions < 1) return fm_fail(FM_BAD_ARG, "fm_build: need >= 1 action");
    if (h->hx < 0 || h->hy < 0) return fm_fail(FM_BAD_ARG, "fm_build: negative sub-grid");
    const long long nslot = (long long)(2 * h->hx + 1) * (2 * h->hy + 1);
    if (nslot + 1 > 65535) return fm_fail(FM_BAD_ARG, "fm_build: sub-grid too large (%lld slots)", nslot);
    if (h->t0 < 0 || h->t1 > G.nt || h->t0 >= h->t1 || h->j0 < 0 || h->j1 > G.ny || h->j0 >= h->j1)
        return fm_fail(FM_BAD_ARG, "fm_build: bad slab/strip range");
    if (M->n_actions != h->n_actions || M->nt != G.nt || M->nx != G.nx || M->ny != G.ny)
        return fm_fail(FM_BAD_ARG, "fm_build: model header does not match the problem");
    if (M->cell0 < 0 || M->ncell < 1 || M->cell0 + M->ncell > G.nx * G.ny ||
        M->n_rows != (int64_t)G.nt * M->ncell * h->n_actions)
        return fm_fail(FM_BAD_ARG, "fm_build: model rows do not match its cell range");
    if (h->j0 * G.nx < M->cell0 || h->j1 * G.nx > M->cell0 + M->ncell)
        return fm_fail(FM_BAD_ARG, "fm_build: rows [%d, %d) are outside the model's cells", h->j0, h->j1);
    if (h->reward.target_i < 0 || h->reward.target_i >= G.nx || h->reward.target_j < 0 || h->reward.target_j >= G.ny)
        return fm_fail(FM_BAD_ARG, "target cell (%d, %d) outside grid", h->reward.target_i, h->reward.target_j);

    K = BuildK{};
    K.nx = G.nx; K.ny = G.ny; K.nt = G.nt; K.nc = G.nx * G.ny;
    K.dx = G.dx; K.dt = G.dt; K.ox = G.ox; K.oy = G.oy;
    K.inv_dx = 1.0 / G.dx;
    K.half_dx = 0.5 * G.dx;   // `0.5 * grid.dx` (environment.py:356)
    K.inv_half_dx = 1.0 / K.half_dx;   // exact for a power-of-two dx (the only case it is used)
    K.dev_flags = getenv("FM_DEV_FLAGS") ? atoi(getenv("FM_DEV_FLAGS")) : 0;
    K.mean = h->env.mean; K.modes = h->env.modes; K.coeffs = h->env.coeffs; K.g = h->env.g;
    K.mask = h->env.mask; K.sat = h->mask_sat;
    K.nm = h->env.n_modes; K.nr = h->env.n_real;
    K.act = h->actions; K.na = h->n_actions; K.obj = h->reward.objective;
    K.h_cr = 0.5 * h->reward.c_r;   // `0.5 * rcfg.c_r` (model_builder.py:358)
    K.r_term = h->reward.r_term; K.r_out = h->reward.r_outbound;
    K.tcell = h->reward.target_j * G.nx + h->reward.target_i;
    K.hx = h->hx; K.hy = h->hy; K.width = 2 * h->hx + 1; K.nslot = (int)nslot;
    K.hw = (int)((nslot + 2) / 2);
    K.rx = h->rx; K.ry = h->ry;
    K.t0 = h->t0; K.t1 = h->t1;
    K.cell0 = h->j0 * G.nx; K.ncell = (h->j1 - h->j0) * G.nx;
    K.AG = h->n_actions < 32 ? h->n_actions : 32;
    K.nag = (h->n_actions + 31) / 32;
    K.CW = 32 / K.AG; if (K.CW < 1) K.CW = 1;
    K.RW = 32 / K.CW;
    K.groups = (K.ncell + K.CW - 1) / K.CW;
    K.n_tasks = (long long)(h->t1 - h->t0) * K.groups * K.nag;
    if (K.n_tasks > 0xFFFFFFF0LL) return fm_fail(FM_BAD_ARG, "fm_build: too many tasks");
    // realizations per chunk: RW recon lanes per cell, 64 realizations
    smem_layout_fit(K, 0, false);
    K.src_cell_exact = source_cells_exact(G) ? 1 : 0;
    K.sx_lo = G.nx;
    K.sx_hi = -1;
    K.sy_lo = G.ny;
    K.sy_hi = -1;
    K.mcell0 = M->cell0; K.mncell = M->ncell;
    K.mcell0 = M->cell0; K.mncell = M->ncell;
    K.reserve_sms = h->reserve_sms > 0 ? h->reserve_sms : 0;
    K.row_ptr = M->row_ptr; K.row_nnz = M->row_nnz; K.reward = M->reward;
    K.entries = M->entries; K.capacity = M->capacity;
    K.nnz_counter = reinterpret_cast<unsigned long long *>(M->d_nnz);
    K.viol = h->viol_flags; K.task_counter = h->task_counter;

    flags = 0;
    if (G.dt == 1.0) flags |= F_DT_ONE;
    if (G.ox == 0.0 && G.oy == 0.0) flags |= F_OX_ZERO;
    if (G.dx == 1.0) flags |= F_DX_ONE;
    else if (is_pow2(G.dx)) flags |= F_DX_MUL;
    if (K.obj == FM_OBJ_NET_ENERGY) flags |= F_NET;

    K.gate_r = h->d_gate_r;
    if (h->h_actions && prove_lean(h)) {
        flags |= F_PROVEN;
        double ax = 0.0, ay = 0.0;
        for (int a = 0; a < h->n_actions; ++a) {
            ax = fmax(ax, fabs(h->h_actions[a].ax));
            ay = fmax(ay, fabs(h->h_actions[a].ay));
        }
        // reach bound of prove_lean, widened by a relative 2^-40 for the
        // rounding of x0 + p (|fl(x0 + p) - (x0 + p)| <= ulp)
        const double mx = fmax(fabs(G.ox), fabs(G.ox + G.nx * G.dx)), my = fmax(fabs(G.oy), fabs(G.oy + G.ny * G.dx));
        const double Rx = (h->vmax_x + ax) * G.dt * (1.0 + 0x1p-40) + 0x1p-40 * mx;
        const double Ry = (h->vmax_y + ay) * G.dt * (1.0 + 0x1p-40) + 0x1p-40 * my;
        sterbenz_axis(G.nx, G.ox, G.dx, Rx, K.sx_lo, K.sx_hi);
        sterbenz_axis(G.ny, G.oy, G.dx, Ry, K.sy_lo, K.sy_hi);
        if ((K.obj != FM_OBJ_NET_ENERGY && rewards_sum_exactly(h)) || h->reward_mode == 1) flags |= F_CNT;
    }
    if (K.smem_warp > smem_block_optin()) {
        // the shared histogram does not fit even one warp: global fallback
        smem_layout(K, K.RW >= 32 ? K.RW : 32, 0, false, true);
        flags = (flags & F_NET) | F_GHIST;
    }
    if ((flags & F_PROVEN) && (flags & F_CNT) && !(flags & F_GHIST) && !getenv("FM_NO_BINS")) {
        bin_params(h, K);
        if (K.bin_ok && K.off_block + K.smem_warp > smem_block_optin()) {   // no room: per transition
            K.bin_ok = 0;
            K.off_block = 0;
            smem_layout_fit(K, 0, false);
        }
    }
    return FM_OK;
}

// Bin path inputs for slabs [t0, t1): f32 coefficients padded to 8 modes
// ([t - t0][r][8]) and max_r |coeff| per (t, m) (the error bound's T).
// Bin path inputs for slabs [t0, t1): f32 coefficients padded to 8 modes
// and to nr_pad realizations ([t - t0][r][8]) and max_r |coeff| per (t, m)
// (the error bound's T).  Block (chunk, t): a grid-stride pass, then one
// block-level max per mode (8 atomics per block, NaN-sticky).
__global__ void __launch_bounds__(256) k_bin_prep(const double *coeffs, int t0, int nts, int nr, int nr_pad, int nm,
                                                  float *c32, double *cmax)
{
    const int tl = blockIdx.y;
    const double *base = coeffs + (size_t)(t0 + tl) * nr * nm;
    double mx[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) mx[m] = 0.0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nr_pad; r += gridDim.x * blockDim.x) {
        float out[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const double c = (m < nm && r < nr) ? base[(size_t)r * nm + m] : 0.0;
            out[m] = (float)c;
            mx[m] = nan_max(mx[m], fabs(c));
        }
        float4 *dst = reinterpret_cast<float4 *>(c32 + ((size_t)tl * nr_pad + r) * 8);
        dst[0] = make_float4(out[0], out[1], out[2], out[3]);
        dst[1] = make_float4(out[4], out[5], out[6], out[7]);
    }
    __shared__ double red[8][8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const double w = warp_max_f64(mx[m]);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][m] = w;
    }
    __syncthreads();
    if (threadIdx.x < nm && threadIdx.x < 8) {
        double w = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) w = nan_max(w, red[k][threadIdx.x]);
        // non-negative doubles (and +NaN) order like their bit patterns
        atomicMax(reinterpret_cast<unsigned long long *>(cmax + (size_t)tl * nm + threadIdx.x),
                  (unsigned long long)__double_as_longlong(w));
    }
}

extern "C" int32_t fm_build_launch(const fm_build_args *h, fm_model *M, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    BuildK K;
    int flags = 0;
    int32_t st = build_params(h, M, K, flags);
    if (st != FM_OK) return st;
    st = frac_table_init();
    if (st != FM_OK) return st;
    FM_CK(cudaMemsetAsync(h->task_counter, 0, sizeof(unsigned int), s));
    float *c32 = nullptr;
    double *cmax = nullptr;
    if (K.bin_ok) {
        const int nts = K.t1 - K.t0;
        // whole iterations of H chunks of 32 (H = 2, or FM_BIN_H with an
        // 8-chunk ring): C2 pads 5000 -> 5056 realizations, not 5120
        constexpr int kPadR = 32 * (FM_BIN_H > 2 ? FM_BIN_H : 2);
        K.nr_pad = (K.nr + kPadR - 1) / kPadR * kPadR;
        FM_CK(cudaMallocAsync(reinterpret_cast<void **>(&c32), sizeof(float) * 8 * (size_t)nts * K.nr_pad, s));
        FM_CK(cudaMallocAsync(reinterpret_cast<void **>(&cmax), sizeof(double) * (size_t)nts * (K.nm ? K.nm : 1), s));
        FM_CK(cudaMemsetAsync(cmax, 0, sizeof(double) * (size_t)nts * (K.nm ? K.nm : 1), s));
        const int bxp = (K.nr_pad + 1023) / 1024;   // 4 realizations per thread
        k_bin_prep<<<dim3(bxp, nts), 256, 0, s>>>(K.coeffs, K.t0, nts, K.nr, K.nr_pad, K.nm, c32, cmax);
        FM_CK_LAUNCH("k_bin_prep");
        K.coef32 = c32;
        K.cmax = cmax;
    }
    st = launch_build(K, flags, (size_t)4 * K.smem_warp, s, (h->phases & 3) ? (h->phases & 3) : 3);
    if (c32) FM_CK(cudaFreeAsync(c32, s));
    if (cmax) FM_CK(cudaFreeAsync(cmax, s));
    return st;
}

extern "C" int32_t fm_build_check(const fm_build_args *h, fm_model *M, uint64_t *h_needed, fm_violation *h_viol,
                                  void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    BuildK K;
    int flags = 0;
    int32_t st = build_params(h, M, K, flags);
    if (st != FM_OK) return st;
    const fm_grid &G = h->grid;
    // census + violation flags back to the host (the reference raises
    // before returning anything, so the error check is synchronous).
    unsigned long long nnz = 0;
    FM_CK(cudaMemcpyAsync(&nnz, M->d_nnz, sizeof(nnz), cudaMemcpyDeviceToHost, s));
    std::vector<uint32_t> flags_h((size_t)G.nt * h->n_actions);
    FM_CK(cudaMemcpyAsync(flags_h.data(), h->viol_flags, flags_h.size() * 4, cudaMemcpyDeviceToHost, s));
    FM_CK(cudaStreamSynchronize(s));
    for (int t = h->t0; t < h->t1; ++t)
        for (int a = 0; a < h->n_actions; ++a) {
            if (!flags_h[(size_t)t * h->n_actions + a]) continue;
            // reproduce the reference message for the first (t, a)
            unsigned long long *d_best;
            FM_CK(cudaMallocAsync(&d_best, sizeof(unsigned long long) + 2 * sizeof(int32_t), s));
            int32_t *d_didj = reinterpret_cast<int32_t *>(d_best + 1);
            FM_CK(cudaMemsetAsync(d_best, 0, sizeof(unsigned long long) + 2 * sizeof(int32_t), s));
            const long long n = (long long)K.nr * K.nc;
            const unsigned nb = (unsigned)((n + 255) / 256);
            k_viol_report<<<nb, 256, 0, s>>>(K, t, a, 0, d_best, d_didj);
            k_viol_report<<<nb, 256, 0, s>>>(K, t, a, 1, d_best, d_didj);
            FM_CK_LAUNCH_N("k_viol_report", 2);
            int32_t didj[2] = {0, 0};
            FM_CK(cudaMemcpyAsync(didj, d_didj, sizeof(didj), cudaMemcpyDeviceToHost, s));
            FM_CK(cudaFreeAsync(d_best, s));
            FM_CK(cudaStreamSynchronize(s));
            if (h_viol) {
                h_viol->t = t; h_viol->a = a; h_viol->di = didj[0]; h_viol->dj = didj[1];
            }
            return fm_fail(FM_SUBGRID_OVERFLOW,
                           "displacement (%d,%d) at t=%d, a=%d exceeds sub-grid half widths (%d,%d)",
                           didj[0], didj[1], t, a, h->hx, h->hy);
        }
    if (h_needed) *h_needed = nnz;
    if (nnz > M->capacity)
        return fm_fail(FM_CAPACITY, "fm_build: entry capacity %llu < %llu needed",
                       (unsigned long long)M->capacity, nnz);
    return FM_OK;
}

extern "C" int32_t fm_build(const fm_build_args *h, fm_model *M, uint64_t *h_needed, fm_violation *h_viol,
                            void *stream)
{
    int32_t st = fm_build_launch(h, M, stream);
    if (st != FM_OK) return st;
    return fm_build_check(h, M, h_needed, h_viol, stream);
}

// Obstacle-gate radius on the device (model_builder.py:218-223 with the
// triangle bound of environment.py:404-419), same arithmetic as the host:
// per_t = max|mean| (+) sum_m max|coef| (x) max|mode|, bound = max_t per_t,
// r = ceil(((bound + f_max) * dt) / dx) + 1.
__global__ void k_gate_radius(fm_grid G, const double *meanmax, const double *coefmax, const double *modemax, int nm,
                              double f_max, int32_t *out2, double *bound2)
{
    if (threadIdx.x >= 2) return;
    const int c = threadIdx.x;
    double b = 0.0;
    for (int t = 0; t < G.nt; ++t) {
        double per = meanmax[t * 2 + c];
        for (int m = 0; m < nm; ++m) per = DADD(per, DMUL(coefmax[t * nm + m], modemax[(m * G.nt + t) * 2 + c]));
        b = t == 0 ? per : fmax(b, per);
    }
    const double reach = DDIV(DMUL(DADD(b, f_max), G.dt), G.dx);
    out2[c] = (int32_t)ceil(reach) + 1;
    if (bound2) bound2[c] = b;
}

extern "C" int32_t fm_gate_radius(fm_grid G, const double *meanmax, const double *coefmax, const double *modemax,
                                  int32_t n_modes, double f_max, int32_t *d_out2, double *d_bound2, void *stream)
{
    k_gate_radius<<<1, 32, 0, (cudaStream_t)stream>>>(G, meanmax, coefmax, modemax, n_modes, f_max, d_out2, d_bound2);
    FM_CK_LAUNCH("k_gate_radius");
    return FM_OK;
}

// ---------------------------------------------------------------------------
// exclusive scan (u64), three-phase, used by the exporters
// ---------------------------------------------------------------------------
static constexpr int kScanBlock = 1024;   // elements per block (256 thr x 4)

__global__ void k_scan_block(uint64_t *data, int64_t n, uint64_t *block_sums)
{
    __shared__ uint64_t sh[256];
    const int64_t base = (int64_t)blockIdx.x * kScanBlock;
    uint64_t v[4];
    uint64_t sum = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t i = base + threadIdx.x * 4 + k;
        v[k] = i < n ? data[i] : 0;
        sum += v[k];
    }
    sh[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {
        uint64_t y = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
        __syncthreads();
        sh[threadIdx.x] += y;
        __syncthreads();
    }
    uint64_t run = sh[threadIdx.x] - sum;   // exclusive prefix of this thread
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t i = base + threadIdx.x * 4 + k;
        if (i < n) data[i] = run;
        run += v[k];
    }
    if (threadIdx.x == 255 && block_sums) block_sums[blockIdx.x] = sh[255];
}

__global__ void k_scan_add(uint64_t *data, int64_t n, const uint64_t *block_offs)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) data[i] += block_offs[i / kScanBlock];
}

// in-place exclusive scan of data[0..n); returns through data; uses tmp
static int32_t scan_u64(uint64_t *data, int64_t n, cudaStream_t s)
{
    if (n <= 0) return FM_OK;
    const int64_t nb = (n + kScanBlock - 1) / kScanBlock;
    if (nb == 1) {
        k_scan_block<<<1, 256, 0, s>>>(data, n, nullptr);
        FM_CK_LAUNCH("k_scan_block");
        return FM_OK;
    }
    uint64_t *sums = nullptr;
    FM_CK(cudaMallocAsync(&sums, (size_t)nb * sizeof(uint64_t), s));
    k_scan_block<<<(unsigned)nb, 256, 0, s>>>(data, n, sums);
    FM_CK_LAUNCH("k_scan_block");
    int32_t st = scan_u64(sums, nb, s);
    if (st != FM_OK) return st;
    k_scan_add<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(data, n, sums);
    FM_CK_LAUNCH("k_scan_add");
    FM_CK(cudaFreeAsync(sums, s));
    return FM_OK;
}

// ---------------------------------------------------------------------------
// export to canonical COO blocks (model_builder.py:474-501, 568-573)
// ---------------------------------------------------------------------------
struct ModelK {
    int nx, ny, nt, nc, na, nr, hx, hy, width, nslot;
    int cell0, ncell;   // cells whose rows the model holds (row = (t*ncell + c - cell0)*na + a)
    long long n_rows, n_g;
    unsigned long long capacity;
    const uint64_t *row_ptr;
    const uint16_t *row_nnz;
    const double *reward;
    const uint32_t *entries;
};

static ModelK model_k(const fm_model *M)
{
    ModelK K;
    K.nx = M->nx; K.ny = M->ny; K.nt = M->nt; K.nc = M->nx * M->ny; K.na = M->n_actions;
    K.nr = M->n_real; K.hx = M->hx; K.hy = M->hy; K.width = 2 * M->hx + 1;
    K.nslot = (2 * M->hx + 1) * (2 * M->hy + 1);
    K.cell0 = M->cell0; K.ncell = M->ncell;
    K.n_rows = M->n_rows; K.n_g = (long long)M->nt * K.nc;
    K.row_ptr = M->row_ptr; K.row_nnz = M->row_nnz; K.reward = M->reward; K.entries = M->entries;
    K.capacity = M->capacity;
    return K;
}

// counts in (a, t, c) order
__global__ void k_export_count(const ModelK K, uint64_t *cnt)
{
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= K.n_rows) return;
    const long long c = idx % K.nc;
    const long long at = idx / K.nc;
    const long long t = at % K.nt, a = at / K.nt;
    cnt[idx] = K.row_nnz[(t * K.nc + c) * K.na + a];
}

__global__ void k_export_fill(const ModelK K, const uint64_t *off, uint32_t *rows, uint32_t *cols, double *vals,
                              double *rewards, uint64_t *block_off)
{
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= K.n_rows) return;
    const long long c = idx % K.nc;
    const long long at = idx / K.nc;
    const long long t = at % K.nt, a = at / K.nt;
    const long long row = (t * K.nc + c) * K.na + a;
    const long long s = t * K.nc + c;
    rewards[a * K.n_g + s] = K.reward[row];
    if (c == 0) block_off[at] = off[idx];
    if (idx == K.n_rows - 1) block_off[(long long)K.na * K.nt] = off[idx] + K.row_nnz[row];
    uint64_t pos = off[idx];
    const uint64_t p = K.row_ptr[row];
    const int n = K.row_nnz[row];
    const int ci = (int)(c % K.nx), cj = (int)(c / K.nx);
    for (int k = 0; k < n; ++k) {
        const uint32_t e = K.entries[p + k];
        const int slot = (int)(e >> 16);
        const uint32_t count = e & 0xffffu;
        uint32_t col;
        if (slot == K.nslot) {
            col = (uint32_t)K.n_g;
        } else {
            const int dj = slot / K.width - K.hy, di = slot % K.width - K.hx;
            col = (uint32_t)((t + 1) * K.nc + (long long)(cj + dj) * K.nx + (ci + di));
        }
        rows[pos] = (uint32_t)s;
        cols[pos] = col;
        vals[pos] = DDIV((double)count, (double)K.nr);   // model_builder.py:491
        ++pos;
    }
}

extern "C" int32_t fm_export_coo(const fm_model *M, uint64_t *d_scratch, uint64_t *d_block_off, uint32_t *rows,
                                 uint32_t *cols, double *vals, double *rewards, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    const ModelK K = model_k(M);
    if (K.n_rows <= 0) return fm_fail(FM_BAD_ARG, "fm_export_coo: empty model");
    if (K.cell0 != 0 || K.ncell != K.nc)
        return fm_fail(FM_BAD_ARG, "fm_export_coo: needs a model of whole layers (this one holds a row strip)");
    const unsigned nb = (unsigned)((K.n_rows + 255) / 256);
    k_export_count<<<nb, 256, 0, s>>>(K, d_scratch);
    FM_CK_LAUNCH("k_export_count");
    int32_t st = scan_u64(d_scratch, K.n_rows, s);
    if (st != FM_OK) return st;
    k_export_fill<<<nb, 256, 0, s>>>(K, d_scratch, rows, cols, vals, rewards, d_block_off);
    FM_CK_LAUNCH("k_export_fill");
    return FM_OK;
}

// ---------------------------------------------------------------------------
// K_solve: backward Bellman layer over the compact model
// ---------------------------------------------------------------------------
struct SolveK {
    ModelK M;
    int t, cell0, ncell;
    int CW, AG, nag, groups;
    const double *ptab;   // ptab[count] = count / n_real
    double *V;
    uint16_t *pi;
};

__global__ void k_prob_table(double *ptab, int nr)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k <= nr) ptab[k] = DDIV((double)k, (double)nr);
}

#ifndef FM_SOLVE_PDL
#define FM_SOLVE_PDL 1
#endif

__global__ void __launch_bounds__(256) k_solve_layer(const SolveK S)
{
    extern __shared__ int soff[];   // slot -> dj*nx + di
    const ModelK &K = S.M;
#if FM_SOLVE_PDL
    // programmatic dependent launch: the next layer's blocks may be scheduled
    // now; they run their prologue and then wait (griddepcontrol.wait) for
    // this grid to complete and its V / policy writes to be visible
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    for (int k = threadIdx.x; k < K.nslot; k += blockDim.x)
        soff[k] = (k / K.width - K.hy) * K.nx + (k % K.width - K.hx);
#if FM_SOLVE_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");   // nothing above reads device data
#endif
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int grp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (grp >= S.groups) return;
    const int cs = lane / S.AG, a_loc = lane - (lane / S.AG) * S.AG;
    const int lc = grp * S.CW + cs;
    const bool cell_ok = lane < S.CW * S.AG && lc < S.ncell;
    const int c = S.cell0 + lc;
    const int t = S.t;
    const double *Vn = S.V + (size_t)(t + 1) * K.nc + c;   // only dereferenced for non-OUT slots
    const double vsink = S.V[K.n_g];
    double best = 0.0;
    int best_a = -1;
    for (int ag = 0; ag < S.nag; ++ag) {
        const int a = ag * 32 + a_loc;
        if (cell_ok && a < K.na) {
            const size_t row = ((size_t)t * K.ncell + (c - K.cell0)) * K.na + a;
            const uint64_t p = K.row_ptr[row];
            // an over-capacity build (deferred check) is discarded; never read past the buffer
            const int n = p + K.row_nnz[row] <= K.capacity ? K.row_nnz[row] : 0;
            double acc = 0.0;   // np.bincount starts every row at +0.0
            for (int k = 0; k < n; ++k) {
                const uint32_t e = __ldg(K.entries + p + k);
                const int slot = (int)(e >> 16);
                const double pr = __ldg(S.ptab + (e & 0xffffu));
                const double vv = slot == K.nslot ? vsink : __ldg(Vn + soff[slot]);
                acc = DADD(acc, DMUL(pr, vv));
            }
            const double q = DADD(K.reward[row], acc);   // q[a] = R + bincount (solver.py:69-71)
            if (best_a < 0 || q > best) {
                best = q;
                best_a = a;
            }
        }
    }
    // first maximum across the AG lanes of this cell (np.argmax semantics)
    for (int o = 1; o < 32; o <<= 1) {
        const double ob = __shfl_down_sync(kFull, best, o);
        const int oa = __shfl_down_sync(kFull, best_a, o);
        const bool same_cell = (a_loc + o) < S.AG && lane + o < 32;
        if (same_cell && oa >= 0 && (best_a < 0 || ob > best || (ob == best && oa < best_a))) {
            best = ob;
            best_a = oa;
        }
    }
    if (cell_ok && a_loc == 0 && best_a >= 0) {
        S.V[(size_t)t * K.nc + c] = best;
        S.pi[(size_t)t * K.nc + c] = (uint16_t)best_a;
    }
}

static int32_t solve_layer(const fm_model *M, const double *ptab, int t, int j0, int j1, double *V, uint16_t *pi,
                           cudaStream_t s)
{
    SolveK S;
    S.M = model_k(M);
    S.t = t;
    S.cell0 = j0 * M->nx;
    S.ncell = (j1 - j0) * M->nx;
    if (S.cell0 < M->cell0 || S.cell0 + S.ncell > M->cell0 + M->ncell)
        return fm_fail(FM_BAD_ARG, "solve: rows [%d, %d) are not in the model", j0, j1);
    S.AG = M->n_actions < 32 ? M->n_actions : 32;
    S.nag = (M->n_actions + 31) / 32;
    S.CW = 32 / S.AG;
    if (S.CW < 1) S.CW = 1;
    S.groups = (S.ncell + S.CW - 1) / S.CW;
    S.ptab = ptab;
    S.V = V;
    S.pi = pi;
    const int wpb = 8;
    const unsigned nb = (unsigned)((S.groups + wpb - 1) / wpb);
    const size_t smem = sizeof(int) * (size_t)S.M.nslot;
#if FM_SOLVE_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb);
    cfg.blockDim = dim3(wpb * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t le = cudaLaunchKernelEx(&cfg, k_solve_layer, S);
    if (le != cudaSuccess) return fm_fail(FM_CUDA_ERROR, "launch k_solve_layer: %s", cudaGetErrorString(le));
#else
    k_solve_layer<<<nb, wpb * 32, smem, s>>>(S);
#endif
    FM_CK_LAUNCH("k_solve_layer");
    return FM_OK;
}

static double *prob_table(const fm_model *M, cudaStream_t s, int32_t *st)
{
    double *ptab = nullptr;
    cudaError_t e = cudaMallocAsync(&ptab, sizeof(double) * (size_t)(M->n_real + 1), s);
    if (e != cudaSuccess) {
        *st = fm_fail(FM_CUDA_ERROR, "cudaMallocAsync: %s", cudaGetErrorString(e));
        return nullptr;
    }
    k_prob_table<<<(M->n_real + 256) / 256, 256, 0, s>>>(ptab, M->n_real);
    g_launches += 1;
    e = cudaGetLastError();
    *st = e == cudaSuccess ? FM_OK : fm_fail(FM_CUDA_ERROR, "launch k_prob_table: %s", cudaGetErrorString(e));
    return ptab;
}

extern "C" int32_t fm_solve_backward(const fm_model *M, int32_t t_lo, int32_t t_hi, double *values,
                                     uint16_t *policy, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    if (t_lo < 0 || t_hi > M->nt || t_lo >= t_hi) return fm_fail(FM_BAD_ARG, "fm_solve_backward: bad t range");
    int32_t st;
    double *ptab = prob_table(M, s, &st);
    if (st != FM_OK) return st;
    if (M->ncell % M->nx || M->cell0 % M->nx) return fm_fail(FM_BAD_ARG, "fm_solve_backward: model strip not whole rows");
    for (int t = t_hi - 1; t >= t_lo; --t) {
        st = solve_layer(M, ptab, t, M->cell0 / M->nx, (M->cell0 + M->ncell) / M->nx, values, policy, s);
        if (st != FM_OK) return st;
    }
    FM_CK(cudaFreeAsync(ptab, s));
    return FM_OK;
}

extern "C" int32_t fm_solve_backward_halo(const fm_model *M, int32_t t_lo, int32_t t_hi, double *values,
                                          uint16_t *policy, fm_halo_fn halo, void *user, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    if (t_lo < 0 || t_hi > M->nt || t_lo >= t_hi) return fm_fail(FM_BAD_ARG, "fm_solve_backward_halo: bad t range");
    if (M->ncell % M->nx || M->cell0 % M->nx)
        return fm_fail(FM_BAD_ARG, "fm_solve_backward_halo: model strip not whole rows");
    int32_t st;
    double *ptab = prob_table(M, s, &st);
    if (st != FM_OK) return st;
    const int j0 = M->cell0 / M->nx, j1 = (M->cell0 + M->ncell) / M->nx;
    for (int t = t_hi - 1; t >= t_lo; --t) {
        st = solve_layer(M, ptab, t, j0, j1, values, policy, s);
        if (st == FM_OK && halo && halo(user, t, stream) != 0)
            st = fm_fail(FM_BAD_ARG, "fm_solve_backward_halo: halo hook failed at layer %d", t);
        if (st != FM_OK) {
            cudaFreeAsync(ptab, s);
            return st;
        }
    }
    FM_CK(cudaFreeAsync(ptab, s));
    return FM_OK;
}

extern "C" int32_t fm_solve_layer(const fm_model *M, int32_t t, int32_t j0, int32_t j1, double *values,
                                  uint16_t *policy, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    if (t < 0 || t >= M->nt || j0 < 0 || j1 > M->ny || j0 >= j1)
        return fm_fail(FM_BAD_ARG, "fm_solve_layer: bad range");
    int32_t st;
    double *ptab = prob_table(M, s, &st);
    if (st != FM_OK) return st;
    st = solve_layer(M, ptab, t, j0, j1, values, policy, s);
    if (st != FM_OK) return st;
    FM_CK(cudaFreeAsync(ptab, s));
    return FM_OK;
}

extern "C" int32_t fm_prob_table(int32_t n_real, double *d_ptab, void *stream)
{
    if (n_real < 1 || !d_ptab) return fm_fail(FM_BAD_ARG, "fm_prob_table: bad arguments");
    k_prob_table<<<(n_real + 256) / 256, 256, 0, (cudaStream_t)stream>>>(d_ptab, n_real);
    FM_CK_LAUNCH("k_prob_table");
    return FM_OK;
}

extern "C" int32_t fm_solve_layer_tab(const fm_model *M, const double *d_ptab, int32_t t, int32_t j0, int32_t j1,
                                      double *values, uint16_t *policy, void *stream)
{
    if (t < 0 || t >= M->nt || j0 < 0 || j1 > M->ny || j0 >= j1 || !d_ptab)
        return fm_fail(FM_BAD_ARG, "fm_solve_layer_tab: bad range");
    return solve_layer(M, d_ptab, t, j0, j1, values, policy, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// general CSR path (host-supplied SparseModel): Jacobi VI, greedy, policy
// ---------------------------------------------------------------------------
__global__ void k_csr_count(const uint32_t *rows, const int64_t *seg_off, int na, int64_t n_g, uint64_t *cnt,
                            int32_t *sorted)
{
    const int a = blockIdx.y;
    const int64_t lo = seg_off[a], hi = seg_off[a + 1];
    for (int64_t k = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < hi; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = rows[k];
        if ((int64_t)r >= n_g) {
            *sorted = 0;
            continue;
        }
        atomicAdd(reinterpret_cast<unsigned long long *>(cnt + (int64_t)a * n_g + r), 1ull);
        if (k > lo && rows[k - 1] > r) *sorted = 0;
    }
}

extern "C" int32_t fm_csr_row_ptr(const uint32_t *rows, const int64_t *h_seg_off, int32_t na, int64_t n_g,
                                  int64_t *row_ptr, int32_t *d_sorted_flag, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = (int64_t)na * n_g + 1;
    FM_CK(cudaMemsetAsync(row_ptr, 0, sizeof(int64_t) * n, s));
    int64_t *d_off = nullptr;
    FM_CK(cudaMallocAsync(&d_off, sizeof(int64_t) * (na + 1), s));
    FM_CK(cudaMemcpyAsync(d_off, h_seg_off, sizeof(int64_t) * (na + 1), cudaMemcpyHostToDevice, s));
    const int one = 1;
    FM_CK(cudaMemcpyAsync(d_sorted_flag, &one, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    dim3 grid(64, na);
    k_csr_count<<<grid, 256, 0, s>>>(rows, d_off, na, n_g, reinterpret_cast<uint64_t *>(row_ptr), d_sorted_flag);
    FM_CK_LAUNCH("k_csr_count");
    int32_t st = scan_u64(reinterpret_cast<uint64_t *>(row_ptr), n, s);
    if (st != FM_OK) return st;
    FM_CK(cudaFreeAsync(d_off, s));
    FM_CK(cudaStreamSynchronize(s));   // h_seg_off / `one` are host stack memory
    return FM_OK;
}

struct CsrK {
    int64_t n_g;
    int na;
    const int64_t *rp;
    const uint32_t *cols;
    const double *vals;
    const double *R;
};

__device__ __forceinline__ double csr_q(const CsrK &C, int a, int64_t s, const double *v)
{
    const int64_t lo = C.rp[(int64_t)a * C.n_g + s], hi = C.rp[(int64_t)a * C.n_g + s + 1];
    double acc = 0.0;
    for (int64_t k = lo; k < hi; ++k) acc = DADD(acc, DMUL(C.vals[k], v[C.cols[k]]));
    return DADD(C.R[(int64_t)a * C.n_g + s], acc);
}

// mode 0: v_out = max_a Q (Jacobi sweep); mode 1: fixed policy.
// Residual = max |v_out - v_in| over all n_g + 1 entries; the last block
// decides convergence (solver.py:95-99) so no host round trip is needed.
struct JacK {
    CsrK C;
    const uint16_t *policy;
    int mode;
    double eps;
    unsigned long long *res;       // [max_iter] residual bits
    unsigned int *done_blocks;     // [max_iter]
    int *done;                     // [1]
    unsigned long long *stats;     // [2] iterations, residual bits
};

__global__ void __launch_bounds__(256) k_jacobi(const JacK J, int iter, const double *v_in, double *v_out)
{
    if (*((volatile int *)J.done)) return;
    const CsrK &C = J.C;
    double local = 0.0;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s <= C.n_g;
         s += (int64_t)gridDim.x * blockDim.x) {
        double vn;
        if (s == C.n_g) {
            vn = 0.0;
        } else if (J.mode == 0) {
            vn = csr_q(C, 0, s, v_in);
            for (int a = 1; a < C.na; ++a) {
                const double q = csr_q(C, a, s, v_in);
                if (q > vn) vn = q;
            }
        } else {
            vn = csr_q(C, J.policy[s], s, v_in);
        }
        v_out[s] = vn;
        const double d = fabs(DSUB(vn, v_in[s]));
        local = (d > local || d != d) ? d : local;
    }
    // block max of non-negative (or NaN) bit patterns
    unsigned long long b = (unsigned long long)__double_as_longlong(local);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(kFull, b, o);
        b = y > b ? y : b;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(J.res + iter, b);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned ticket = atomicAdd(J.done_blocks + iter, 1u);
        if (ticket == gridDim.x - 1) {
            __threadfence();
            const unsigned long long rb = atomicAdd(J.res + iter, 0ull);
            const double r = __longlong_as_double((long long)rb);
            J.stats[0] = (unsigned long long)(iter + 1);
            J.stats[1] = rb;
            if (r < J.eps) *J.done = 1;
        }
    }
}

static CsrK csr_k(const fm_csr *h)
{
    CsrK C;
    C.n_g = h->n_g; C.na = h->n_actions; C.rp = h->row_ptr; C.cols = h->cols; C.vals = h->vals; C.R = h->rewards;
    return C;
}

static int32_t run_jacobi(const fm_csr *h, const uint16_t *policy, int mode, double eps, int max_iter, double *v0,
                          double *v1, uint64_t *d_stats, cudaStream_t s)
{
    if (max_iter < 1) return fm_fail(FM_BAD_ARG, "max_iterations must be >= 1");
    JacK J;
    J.C = csr_k(h);
    J.policy = policy;
    J.mode = mode;
    J.eps = eps;
    const size_t scratch = sizeof(unsigned long long) * max_iter + sizeof(unsigned int) * max_iter + sizeof(int) * 4;
    unsigned char *buf = nullptr;
    FM_CK(cudaMallocAsync(&buf, scratch, s));
    FM_CK(cudaMemsetAsync(buf, 0, scratch, s));
    J.res = reinterpret_cast<unsigned long long *>(buf);
    J.done_blocks = reinterpret_cast<unsigned int *>(buf + sizeof(unsigned long long) * max_iter);
    J.done = reinterpret_cast<int *>(buf + sizeof(unsigned long long) * max_iter + sizeof(unsigned int) * max_iter);
    J.stats = reinterpret_cast<unsigned long long *>(d_stats);
    FM_CK(cudaMemsetAsync(d_stats, 0, 2 * sizeof(uint64_t), s));
    FM_CK(cudaMemsetAsync(v0, 0, sizeof(double) * (size_t)(h->n_g + 1), s));
    const int64_t n = h->n_g + 1;
    int nb = (int)((n + 255) / 256);
    const int cap = 8 * sm_count();
    if (nb > cap) nb = cap;
    for (int it = 0; it < max_iter; ++it) {
        const double *vin = (it & 1) ? v1 : v0;
        double *vout = (it & 1) ? v0 : v1;
        k_jacobi<<<nb, 256, 0, s>>>(J, it, vin, vout);
    }
    FM_CK_LAUNCH_N("k_jacobi", max_iter);
    FM_CK(cudaFreeAsync(buf, s));
    return FM_OK;
}

extern "C" int32_t fm_jacobi(const fm_csr *h, double epsilon, int32_t max_iter, double *v0, double *v1,
                             uint64_t *d_stats, void *stream)
{
    return run_jacobi(h, nullptr, 0, epsilon, max_iter, v0, v1, d_stats, (cudaStream_t)stream);
}

extern "C" int32_t fm_policy_value(const fm_csr *h, const uint16_t *policy, double epsilon, int32_t max_iter,
                                   double *v0, double *v1, uint64_t *d_stats, void *stream)
{
    return run_jacobi(h, policy, 1, epsilon, max_iter, v0, v1, d_stats, (cudaStream_t)stream);
}

__global__ void k_greedy(const CsrK C, const double *v, uint16_t *act)
{
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= C.n_g) return;
    double best = csr_q(C, 0, s, v);
    int ba = 0;
    for (int a = 1; a < C.na; ++a) {
        const double q = csr_q(C, a, s, v);
        if (q > best) {
            best = q;
            ba = a;
        }
    }
    act[s] = (uint16_t)ba;
}

extern "C" int32_t fm_greedy(const fm_csr *h, const double *values, uint16_t *actions, void *stream)
{
    const CsrK C = csr_k(h);
    if (C.n_g <= 0) return FM_OK;
    k_greedy<<<(unsigned)((C.n_g + 255) / 256), 256, 0, (cudaStream_t)stream>>>(C, values, actions);
    FM_CK_LAUNCH("k_greedy");
    return FM_OK;
}

// ---------------------------------------------------------------------------
// FP64 pipe probe (roofline denominator)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_fp64_probe(double *sink, int iters)
{
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = 1.0 + 1e-9 * (threadIdx.x + k);
    const double m = 0.999999999, b = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = DADD(DMUL(x[k], m), b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) sink[0] = s;
}

extern "C" int32_t fm_fp64_probe(double *d_sink, int32_t blocks, int32_t iters, void *stream)
{
    k_fp64_probe<<<blocks, 256, 0, (cudaStream_t)stream>>>(d_sink, iters);
    FM_CK_LAUNCH("k_fp64_probe");
    return FM_OK;
}

// ---------------------------------------------------------------------------
// Model file image (io.write_model, io.py:213-244): after fm_export_coo the
// canonical COO sits in block order; one thread per entry writes its row,
// column and f32 probability into the block's three arrays, and one thread
// per (action, state) writes the f32 reward.  The caller writes the header
// (magic, version, sizes, block offsets) in front: `header` bytes.
// ---------------------------------------------------------------------------
__global__ void k_model_image(const uint64_t *block_off, int n_blocks, const uint32_t *rows, const uint32_t *cols,
                              const double *vals, uint64_t nnz, const double *rewards, uint64_t n_rew,
                              uint64_t header, unsigned char *img)
{
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < nnz) {
        int lo = 0, hi = n_blocks - 1;   // block of entry e: last k with block_off[k] <= e
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (block_off[mid] <= e) lo = mid;
            else hi = mid - 1;
        }
        const uint64_t b0 = block_off[lo], n = block_off[lo + 1] - b0, i = e - b0;
        unsigned char *base = img + header + 12 * b0;
        reinterpret_cast<uint32_t *>(base)[i] = rows[e];
        reinterpret_cast<uint32_t *>(base + 4 * n)[i] = cols[e];
        reinterpret_cast<float *>(base + 8 * n)[i] = __double2float_rn(vals[e]);   // astype("<f4")
    }
    if (e < n_rew) reinterpret_cast<float *>(img + header + 12 * nnz)[e] = __double2float_rn(rewards[e]);
}

extern "C" int32_t fm_model_image(const uint64_t *d_block_off, int32_t n_blocks, const uint32_t *rows,
                                  const uint32_t *cols, const double *vals, uint64_t nnz, const double *rewards,
                                  uint64_t n_rewards, uint64_t header_bytes, unsigned char *d_img, void *stream)
{
    if (n_blocks < 1 || (header_bytes & 3)) return fm_fail(FM_BAD_ARG, "fm_model_image: bad layout");
    const uint64_t n = nnz > n_rewards ? nnz : n_rewards;
    if (n == 0) return FM_OK;
    k_model_image<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        d_block_off, n_blocks, rows, cols, vals, nnz, rewards, n_rewards, header_bytes, d_img);
    FM_CK_LAUNCH("k_model_image");
    return FM_OK;
}

// ---------------------------------------------------------------------------
// Ensemble rollout (rollout.py:107-208): one thread per trajectory follows
// the policy through its realization's flow, one step_flat per time index
// (model_builder.py:286-369, want_cause) with the velocity of
// reconstruct_at (environment.py:301-320).  Rows are recorded as (cell,
// action, cause, reward, cumulative reward); the host formats them.
// ---------------------------------------------------------------------------
enum : int { C_MOVE = 0, C_TARGET = 1, C_OUTSIDE = 2, C_HORIZON = 3, C_LAND = 4, C_TRANSIT = 5 };

struct RollK {
    BuildK B;
    const uint16_t *policy;
    int si, sj;
    const int32_t *real;
    int n_traj, max_rows;
    int32_t *row_cell;
    int16_t *row_action;
    int8_t *row_cause;
    double *row_reward, *row_cum;
    int32_t *n_rows, *final_cell;
};

__global__ void __launch_bounds__(128) k_rollout(const __grid_constant__ RollK R)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= R.n_traj) return;
    const BuildK &K = R.B;
    const int r = R.real[k];
    const int rx = K.gate_r ? K.gate_r[0] : K.rx, ry = K.gate_r ? K.gate_r[1] : K.ry;
    int cell = R.sj * K.nx + R.si;
    double cum = 0.0;
    int n = 0, fin = -1;
    const size_t o = (size_t)k * R.max_rows;
    for (int t = 0; t < K.nt; ++t) {
        const int a = R.policy[(size_t)t * K.nc + cell];
        const int ci = cell % K.nx, cj = cell / K.nx;
        const fm_action A = K.act[a];
        int cause, succ = 0;
        double rw;
        bool terminal;
        if (t + 1 >= K.nt) {   // horizon (model_builder.py:319-328)
            cause = C_HORIZON;
            rw = K.r_out;
            terminal = true;
        } else {
            double vx = K.mean[((size_t)t * K.nc + cell) * 2], vy = K.mean[((size_t)t * K.nc + cell) * 2 + 1];
            for (int m = 0; m < K.nm; ++m) {
                const double c = K.coeffs[((size_t)t * K.nr + r) * K.nm + m];
                const double *md = K.modes + (((size_t)m * K.nt + t) * K.nc + cell) * 2;
                vx = DADD(vx, DMUL(c, md[0]));
                vy = DADD(vy, DMUL(c, md[1]));
            }
            const double x0 = DADD(K.ox, DMUL(DADD((double)ci, 0.5), K.dx));   // environment.py:96-103
            const double y0 = DADD(K.oy, DMUL(DADD((double)cj, 0.5), K.dx));
            const double x1 = DADD(x0, DMUL(DADD(vx, A.ax), K.dt)), y1 = DADD(y0, DMUL(DADD(vy, A.ay), K.dt));
            const int i1 = __double2int_rd(to_cell<0>(x1, K.ox, K.dx, K.inv_dx));
            const int j1 = __double2int_rd(to_cell<0>(y1, K.oy, K.dx, K.inv_dx));
            const bool inb = (unsigned)i1 < (unsigned)K.nx && (unsigned)j1 < (unsigned)K.ny;
            succ = inb ? j1 * K.nx + i1 : 0;
            const bool landed = inb && K.mask[(size_t)(t + 1) * K.nc + succ] != 0;
            bool blocked = false;
            if (box_count(K, t, ci - rx, ci + rx, cj - ry, cj + ry) > 0) blocked = seg_blocked<0>(K, t, x0, y0, x1, y1);
            const bool bad = !inb || landed || blocked;
            const bool hit = inb && !bad && succ == K.tcell;
            if (K.obj == FM_OBJ_NET_ENERGY) {
                const double gs = K.g[(size_t)t * K.nc + cell];
                const double gd = inb ? K.g[(size_t)(t + 1) * K.nc + succ] : 0.0;
                const double b = DMUL(DADD(DADD(A.neg_cff, DMUL(K.h_cr, gs)), DMUL(K.h_cr, gd)), K.dt);
                rw = hit ? DADD(b, K.r_term) : b;
            } else {
                rw = hit ? A.base_hit : A.base;
            }
            if (bad) rw = K.r_out;
            cause = hit ? C_TARGET : C_MOVE;   // precedence of model_builder.py:363-366
            if (blocked) cause = C_TRANSIT;
            if (landed) cause = C_LAND;
            if (!inb) cause = C_OUTSIDE;
            terminal = bad;
        }
        cum = DADD(cum, rw);   // cum += reward (rollout.py:148)
        R.row_cell[o + n] = cell;
        R.row_action[o + n] = (int16_t)a;
        R.row_cause[o + n] = (int8_t)cause;
        R.row_reward[o + n] = rw;
        R.row_cum[o + n] = cum;
        ++n;
        if (cause == C_TARGET) {
            fin = succ;
            break;
        }
        if (terminal) break;
        cell = succ;
    }
    R.n_rows[k] = n;
    R.final_cell[k] = fin;
}

extern "C" int32_t fm_rollout(const fm_rollout_args *h, void *stream)
{
    const fm_grid &G = h->grid;
    if (G.nx < 1 || G.ny < 1 || G.nt < 1 || h->n_actions < 1 || h->n_traj < 0 || h->max_rows < G.nt)
        return fm_fail(FM_BAD_ARG, "fm_rollout: bad arguments");
    if (h->start_i < 0 || h->start_i >= G.nx || h->start_j < 0 || h->start_j >= G.ny)
        return fm_fail(FM_BAD_ARG, "start cell (%d, %d) outside grid", h->start_i, h->start_j);
    if (h->n_traj == 0) return FM_OK;
    RollK R{};
    BuildK &K = R.B;
    K = BuildK{};
    K.nx = G.nx; K.ny = G.ny; K.nt = G.nt; K.nc = G.nx * G.ny;
    K.dx = G.dx; K.dt = G.dt; K.ox = G.ox; K.oy = G.oy;
    K.inv_dx = 1.0 / G.dx;
    K.half_dx = 0.5 * G.dx;
    K.mean = h->env.mean; K.modes = h->env.modes; K.coeffs = h->env.coeffs; K.g = h->env.g;
    K.mask = h->env.mask; K.sat = h->mask_sat;
    K.nm = h->env.n_modes; K.nr = h->env.n_real;
    K.act = h->actions; K.na = h->n_actions; K.obj = h->reward.objective;
    K.h_cr = 0.5 * h->reward.c_r;
    K.r_term = h->reward.r_term; K.r_out = h->reward.r_outbound;
    K.tcell = h->reward.target_j * G.nx + h->reward.target_i;
    K.gate_r = h->d_gate_r;
    R.policy = h->policy; R.si = h->start_i; R.sj = h->start_j;
    R.real = h->realizations; R.n_traj = h->n_traj; R.max_rows = h->max_rows;
    R.row_cell = h->row_cell; R.row_action = h->row_action; R.row_cause = h->row_cause;
    R.row_reward = h->row_reward; R.row_cum = h->row_cum; R.n_rows = h->n_rows; R.final_cell = h->final_cell;
    k_rollout<<<(h->n_traj + 127) / 128, 128, 0, (cudaStream_t)stream>>>(R);
    FM_CK_LAUNCH("k_rollout");
    return FM_OK;
}
