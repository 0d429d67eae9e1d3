// decode_stream.cu -- the HBM-streaming schedule of the Min-Sum hot path (steps a2-a7).
//
// One loop body of Alg. 1 over a chunk of frames is two sweeps:
//   k_cn  check-node update, Eq. eta_update through Observations 1 and 2:
//         per row and frame, lambda_e = s_j - eta^prev_e is formed in registers, reduced to
//         (min0, min0Location, min1, sign parity) -- the paper's "four vectors of size m"
//          -- and the sign bit of every lambda_e.  That state IS eta (Eq. etaCalculation,
//         P:327-336, with the delta placement of Obs. 1, reading A2); no per-edge message is stored.
//         Fused: the syndrome of b = slice(s) over the same gathered s.
//   k_bn  bit-node update, Eq. lambda_j / sCalculation: eta_{i,j} rebuilt
//         from the row state, summed over M_j in ascending row order from +0.0, then + r_j (A14).
// The syndrome computed by k_cn at body k is the stopping test of body k-1; k_bn then
// freezes stopped frames and records k-1.  No host round trip anywhere.
//
// Layout: frames are interleaved in tiles of 128 ([tile][row-or-column][128 frames]); lane l of a
// warp owns frames 4l..4l+3 of the tile, so every gather of s, r or row state is one 512-byte
// contiguous float4 access per warp, and per-frame bits of 128 frames are four ballot words.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "ldpc_internal.cuh"

namespace ldpc {

namespace {

constexpr unsigned FULL = 0xffffffffu;

template <typename T>
struct Vec4;
template <>
struct Vec4<uint8_t> {
    using type = uchar4;
};
template <>
struct Vec4<uint16_t> {
    using type = ushort4;
};

__device__ __forceinline__ float comp(const float4 &a, int v) { return v == 0 ? a.x : v == 1 ? a.y : v == 2 ? a.z : a.w; }
__device__ __forceinline__ unsigned comp(const uint4 &a, int v) { return v == 0 ? a.x : v == 1 ? a.y : v == 2 ? a.z : a.w; }
template <typename V>
__device__ __forceinline__ int compl4(const V &a, int v) {
    return v == 0 ? (int)a.x : v == 1 ? (int)a.y : v == 2 ? (int)a.z : (int)a.w;
}

__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ void st4(float *p, float4 v) { *reinterpret_cast<float4 *>(p) = v; }
__device__ __forceinline__ uint4 ldu4(const uint32_t *p) { return *reinterpret_cast<const uint4 *>(p); }

// ------------------------------------------------------------------------------------------------
// a2: stage-in.  llr [F][n] -> r, s [T][n][128] (s = r), init per-tile flags.
// s is stored canonically (-0 -> +0; same slice and same sign() under reading A12), so that the later
// sweeps can read both the decision b = slice(s) and the sign of lambda = s - eta^prev straight from
// IEEE bits: after this no s and no lambda is ever -0 (x - y = -0 only for x = -0 and y = +0, and a
// bit-node sum started at +0.0 is never -0).
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(CTA) k_stage_in(const float *__restrict__ llr, int64_t frames, int n, int T,
                                                  float *__restrict__ r, float *__restrict__ s,
                                                  uint32_t *__restrict__ unsat, uint32_t *__restrict__ done,
                                                  int *__restrict__ fbe, int *__restrict__ fraw, int *__restrict__ fnz,
                                                  int *__restrict__ tcount, int *__restrict__ tlist) {
    __shared__ float tile[32][TILE + 1];
    const int t = blockIdx.y, j0 = blockIdx.x * 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t f0 = (int64_t)t * TILE;
    for (int fl = warp; fl < TILE; fl += CTA / 32) {
        int64_t f = f0 + fl;
        int j = j0 + lane;
        tile[lane][fl] = (f < frames && j < n) ? __ldg(llr + f * n + j) : -1.0f;
    }
    __syncthreads();
    for (int jl = warp; jl < 32; jl += CTA / 32) {
        int j = j0 + jl;
        if (j >= n) break;
        size_t base = ((size_t)t * n + j) * TILE;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            float v = tile[jl][lane + 32 * q];
            r[base + lane + 32 * q] = v;
            s[base + lane + 32 * q] = __fadd_rn(v, 0.0f);  // canonical zero
        }
    }
    if (blockIdx.x == 0) {
        int tid = threadIdx.x;
        if (tid < 4) {
            // frame 4*lane+v of the tile is bit `lane` of word v; padding frames start "done"
            uint32_t pad = 0;
            for (int l = 0; l < 32; l++)
                if (f0 + 4 * l + tid >= frames) pad |= 1u << l;
            done[(size_t)t * 4 + tid] = pad;
            unsat[(size_t)t * 4 + tid] = 0;
            unsat[((size_t)T + t) * 4 + tid] = 0;
        }
        if (tid == 0) {
            tlist[(size_t)T + t] = t;  // body 1 runs every tile
            if (t == 0) {
                tcount[0] = 0;
                tcount[1] = T;
            }
        }
        if (tid < TILE) {
            fbe[(size_t)t * TILE + tid] = 0;
            fraw[(size_t)t * TILE + tid] = 0;
            fnz[(size_t)t * TILE + tid] = 0;
        }
    }
}

// ------------------------------------------------------------------------------------------------
// Encoding of the check-node state (it IS eta: Obs. 1 and 2, reading A2):
//   min0, min1   fp32, both with SIGN BIT = the row's sign parity x (-1)^{d_i} (reading A1), so the
//                magnitude picked by Obs. 1 already carries the row factor of Obs. 2;
//   loc          u8 / u16 min0Location (position inside N_i);
//   sgn          per (tile, edge) four u32 in "ballot layout": bit l of word v is the sign of
//                lambda_e for frame 4l + v -- exactly the four warp ballots the check node produces.
// eta_e = (loc == p ? min1 : min0) with its sign bit XORed with sgn bit: one FSEL and one LOP3 per
// frame-edge; a lane moves its ballot bit to bit 31 with one integer multiply by 2^(31-lane) (FMA
// pipe), which keeps the ALU pipe -- the sweeps' real limiter -- for the min/argmin work.
// ------------------------------------------------------------------------------------------------
template <typename LocT>
struct LocOps;
template <>
struct LocOps<uint8_t> {
    using W = uint32_t;  // the 4 locations of a lane, one byte each
    static __device__ __forceinline__ W load(const uint8_t *p) { return *reinterpret_cast<const uint32_t *>(p); }
    static __device__ __forceinline__ void store(uint8_t *p, const int l[4]) {
        *reinterpret_cast<uint32_t *>(p) =
            (uint32_t)l[0] | ((uint32_t)l[1] << 8) | ((uint32_t)l[2] << 16) | ((uint32_t)l[3] << 24);
    }
    static __device__ __forceinline__ W key(W w, int p) { return w ^ ((uint32_t)p * 0x01010101u); }
    static __device__ __forceinline__ bool hit(W x, int v) { return (x & (0xffu << (8 * v))) == 0u; }
};
template <>
struct LocOps<uint16_t> {
    using W = uint2;
    static __device__ __forceinline__ W load(const uint16_t *p) { return *reinterpret_cast<const uint2 *>(p); }
    static __device__ __forceinline__ void store(uint16_t *p, const int l[4]) {
        *reinterpret_cast<uint2 *>(p) = make_uint2((uint32_t)l[0] | ((uint32_t)l[1] << 16),
                                                   (uint32_t)l[2] | ((uint32_t)l[3] << 16));
    }
    static __device__ __forceinline__ W key(W w, int p) {
        const uint32_t q = (uint32_t)p * 0x00010001u;
        return make_uint2(w.x ^ q, w.y ^ q);
    }
    static __device__ __forceinline__ bool hit(W x, int v) {
        return ((v < 2 ? x.x : x.y) & (0xffffu << (16 * (v & 1)))) == 0u;
    }
};

// the sign of a magnitude picked by Obs. 1 flipped by one stored sign bit (already moved to bit 31)
__device__ __forceinline__ float flip31(float mag, uint32_t bit31) {
    return __uint_as_float(__float_as_uint(mag) ^ (bit31 & 0x80000000u));
}

constexpr int CN_CHUNK = 8;  // edges per sign word and per batch of gathers (4 frames x 8 edges = 32 bits)
#ifndef CN_MINB
#define CN_MINB 2
#endif
#ifndef CN1_MINB
#define CN1_MINB 3
#endif
#ifndef BNL_MINB
#define BNL_MINB 6
#endif
#ifndef CN_T
#define CN_T CTA
#endif
#ifndef BNL_T
#define BNL_T 128  // bit-node CTA size: 128 threads x 12 CTAs per SM measured 1.5-2 % faster than 256 x 6
#endif
#ifndef BNL_COLS
#define BNL_COLS 16
#endif

// ------------------------------------------------------------------------------------------------
// a3/a4/a6: check-node sweep of loop body k (k = 1..L), fused syndrome of b^(k-1).
// FIRST: eta^prev = 0, so no old state is read.
// A warp owns rows i0 + warp + 8q.  Per row, every load -- the d gathers of s (512-byte float4
// segments, lane = 4 frames), the row state and the lane's old sign word -- is issued before any
// arithmetic, and the column indices of the next row are prefetched meanwhile, so each row costs one
// memory latency, overlapped across the warps of the SM.  Per frame-edge: lambda = s_j - eta^prev
// (SEL, LOP3, FADD), first-strict-minimum tracking (FSETP, 3 FMNMX, SEL; reading A13), sign parity
// (LOP3 on the IEEE bits), the new sign bit into the lane's own word, and, when EARLY, the decision
// parity (slice(s) = 0 iff bit 31 of bits(s) - 1 is set, s never -0).
// ------------------------------------------------------------------------------------------------
template <typename LocT, bool FIRST, bool EARLY>
__global__ void __launch_bounds__(CTA, CN_MINB)
    k_cn(Graph g, StreamState w, int k, int rows_per_cta, int literal, const int *kdev) {
    using LO = LocOps<LocT>;
    if (kdev) k = *kdev;  // body index supplied by the graph-driven loop
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t s_u[4];
    // the tiles of body k are the ones with a running frame (list rebuilt by k_bn of body k-1)
    const int cnt = w.tcount[k & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) w.tcount[(k + 1) & 1] = 0;  // rebuilt by k_bn of body k
    if ((int)blockIdx.y >= cnt) return;  // active tiles are compacted to the front of the list
    const int t = w.tlist[(size_t)(k & 1) * w.T + blockIdx.y];
    if (EARLY) {
        if (threadIdx.x < 4) s_u[threadIdx.x] = 0;
        __syncthreads();
    }
    const int m = g.m, n = g.n, wr = g.wr;
    const float *__restrict__ Sl = w.s + (size_t)t * n * TILE + 4 * lane;
    // the tile's row records: [min0 512 B][min1 512 B][loc 128 x sizeof(LocT)][sign words 128 x wr]
    unsigned char *RB = w.rst + (size_t)t * m * w.rs;
    const size_t RSW = (size_t)w.rs / 4, RSL = (size_t)w.rs / sizeof(LocT);  // row strides
    float *__restrict__ M0l = reinterpret_cast<float *>(RB) + 4 * lane;
    float *__restrict__ M1l = reinterpret_cast<float *>(RB) + 128 + 4 * lane;
    LocT *__restrict__ LCl = reinterpret_cast<LocT *>(RB + 1024) + 4 * lane;
    uint32_t *__restrict__ SGl = reinterpret_cast<uint32_t *>(RB + 1024 + 128 * sizeof(LocT)) + lane;
    const float INF = __int_as_float(0x7f800000);
    const int i0 = blockIdx.x * rows_per_cta + warp, i1 = min(m, blockIdx.x * rows_per_cta + rows_per_cta);
    const int nr = i0 < i1 ? (i1 - i0 + 7) / 8 : 0;  // rows of this warp (<= 32)
    int ra = 0, rb = 0;  // lane q: row_ptr of the warp's row q
    if (lane < nr) {
        ra = __ldg(g.row_ptr + i0 + 8 * lane);
        rb = __ldg(g.row_ptr + i0 + 8 * lane + 1);
    }
    int a = __shfl_sync(FULL, ra, 0), d = __shfl_sync(FULL, rb, 0) - a;
    int cj = (nr > 0 && lane < d) ? __ldg(g.col_idx + a + lane) : 0;  // lane q: column of edge q
    uint32_t u0 = 0, u1 = 0, u2 = 0, u3 = 0;
    for (int q = 0; q < nr; q++) {
        const int i = i0 + 8 * q;
        const int an = __shfl_sync(FULL, ra, (q + 1) & 31), dn = __shfl_sync(FULL, rb, (q + 1) & 31) - an;
        const uint32_t corr = (uint32_t)(d & 1) & (uint32_t)(!literal);  // (-1)^{d_i}, reading A1
        float om0[4] = {0.f, 0.f, 0.f, 0.f}, om1[4] = {0.f, 0.f, 0.f, 0.f};
        typename LO::W olc{};
        if (!FIRST) {
            const float4 A = ld4(M0l + (size_t)i * RSW), B = ld4(M1l + (size_t)i * RSW);
            om0[0] = A.x; om0[1] = A.y; om0[2] = A.z; om0[3] = A.w;
            om1[0] = B.x; om1[1] = B.y; om1[2] = B.z; om1[3] = B.w;
            olc = LO::load(LCl + (size_t)i * RSL);
        }
        float nm0[4] = {INF, INF, INF, INF}, nm1[4] = {INF, INF, INF, INF};
        int nloc[4] = {0, 0, 0, 0};
        uint32_t par[4] = {0u, 0u, 0u, 0u}, syn[4] = {0u, 0u, 0u, 0u};
        for (int p0 = 0; p0 < d; p0 += CN_CHUNK) {
            if (p0 > 0 && (p0 & 31) == 0) cj = (lane < d - p0) ? __ldg(g.col_idx + a + p0 + lane) : 0;
            uint32_t *sgp = SGl + (size_t)i * RSW + (p0 >> 3) * 32;
            float4 sv[CN_CHUNK];
#pragma unroll
            for (int u = 0; u < CN_CHUNK; u++) {
                const int j = __shfl_sync(FULL, cj, (p0 + u) & 31);
                sv[u] = ld4(Sl + (size_t)j * TILE);  // unconditional: edges past d_i read column 0
            }
            const uint32_t wold = FIRST ? 0u : *sgp;
            uint32_t wnew = 0;
#pragma unroll
            for (int u = 0; u < CN_CHUNK; u++) {
                if (p0 + u < d) {
                    const int p = p0 + u;
                    typename LO::W key{};
                    if (!FIRST) key = LO::key(olc, p);
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        const float sj = comp(sv[u], v);
                        float x = sj;
                        if (!FIRST) {
                            const float mag = LO::hit(key, v) ? om1[v] : om0[v];  // Obs. 1 (+ row parity)
                            x = sj - flip31(mag, wold << (31 - 4 * u - v));        // lambda_k - eta^prev_{i,k}
                        }
                        const float ax = fabsf(x);
                        const bool lt = ax < nm0[v];  // first strict minimum (A13)
                        nm1[v] = fminf(nm1[v], fmaxf(nm0[v], ax));
                        nm0[v] = fminf(nm0[v], ax);
                        nloc[v] = lt ? p : nloc[v];
                        par[v] ^= __float_as_uint(x);                          // sign parity (Obs. 2)
                        if (EARLY) syn[v] ^= __float_as_uint(sj) - 1u;         // bit 31: slice(s_j) == 0
                        wnew |= (__float_as_uint(x) >> 31) << (4 * u + v);     // sign(0) = +1
                    }
                }
            }
            *sgp = wnew;
        }
        // prefetch the next row's column indices (its state and gathers are issued at its start)
        cj = (q + 1 < nr && lane < dn) ? __ldg(g.col_idx + an + lane) : 0;
        float4 o0, o1;
        {
            const uint32_t c31 = corr << 31;
            const uint32_t s0 = (par[0] & 0x80000000u) ^ c31, s1 = (par[1] & 0x80000000u) ^ c31;
            const uint32_t s2 = (par[2] & 0x80000000u) ^ c31, s3 = (par[3] & 0x80000000u) ^ c31;
            o0 = make_float4(__uint_as_float(__float_as_uint(nm0[0]) | s0), __uint_as_float(__float_as_uint(nm0[1]) | s1),
                             __uint_as_float(__float_as_uint(nm0[2]) | s2), __uint_as_float(__float_as_uint(nm0[3]) | s3));
            o1 = make_float4(__uint_as_float(__float_as_uint(nm1[0]) | s0), __uint_as_float(__float_as_uint(nm1[1]) | s1),
                             __uint_as_float(__float_as_uint(nm1[2]) | s2), __uint_as_float(__float_as_uint(nm1[3]) | s3));
        }
        st4(M0l + (size_t)i * RSW, o0);
        st4(M1l + (size_t)i * RSW, o1);
        LO::store(LCl + (size_t)i * RSL, nloc);
        if (EARLY) {
            const uint32_t dp = (uint32_t)(d & 1);  // XOR_j b_j = d_i mod 2 xor XOR_j (1 - b_j)
            u0 |= __ballot_sync(FULL, ((syn[0] >> 31) ^ dp) != 0u);
            u1 |= __ballot_sync(FULL, ((syn[1] >> 31) ^ dp) != 0u);
            u2 |= __ballot_sync(FULL, ((syn[2] >> 31) ^ dp) != 0u);
            u3 |= __ballot_sync(FULL, ((syn[3] >> 31) ^ dp) != 0u);
        }
        a = an;
        d = dn;
    }
    if (EARLY) {
        if (lane == 0) {
            if (u0) atomicOr(&s_u[0], u0);
            if (u1) atomicOr(&s_u[1], u1);
            if (u2) atomicOr(&s_u[2], u2);
            if (u3) atomicOr(&s_u[3], u3);
        }
        __syncthreads();
        if (threadIdx.x < 4 && s_u[threadIdx.x])
            atomicOr(w.unsat + ((size_t)(k & 1) * w.T + t) * 4 + threadIdx.x, s_u[threadIdx.x]);
    }
}

// ------------------------------------------------------------------------------------------------
// Software-pipelined check-node sweep for codes whose rows all have degree <= CH (<= 8: one sign
// word per row and lane).  Two row buffers in registers: while a warp computes row q from buffer A,
// every load of row q+1 -- its CH gathers of s, its state and its old sign word -- is already in
// flight into buffer B, and the column indices of row q+2 are being fetched.  All loads are
// unconditional (edges past d_i read column 0 of the tile, rows past the warp's last read its first
// row), so the compiler issues them back to back instead of behind predicated moves.
// ------------------------------------------------------------------------------------------------
template <int CH, typename LocT>
struct CnRow {
    float4 sv[CH];
    float4 m0, m1;
    typename LocOps<LocT>::W lc;
    uint32_t wold;
};

template <int CH, typename LocT, bool FIRST>
__device__ __forceinline__ void cn_fetch(CnRow<CH, LocT> &R, int cj, int i, const float *__restrict__ Sl,
                                         const uint32_t *__restrict__ SGl, const float *__restrict__ M0l,
                                         const float *__restrict__ M1l, const LocT *__restrict__ LCl, size_t RSW,
                                         size_t RSL) {
    if (!FIRST) {
        R.wold = SGl[(size_t)i * RSW];
        R.m0 = ld4(M0l + (size_t)i * RSW);
        R.m1 = ld4(M1l + (size_t)i * RSW);
        R.lc = LocOps<LocT>::load(LCl + (size_t)i * RSL);
    }
#pragma unroll
    for (int u = 0; u < CH; u++) {
        const int j = __shfl_sync(FULL, cj, u);
        R.sv[u] = ld4(Sl + (size_t)j * TILE);
    }
}

template <int CH, typename LocT, bool FIRST, bool EARLY>
__device__ __forceinline__ void cn_compute(const CnRow<CH, LocT> &R, int i, int d, int literal,
                                           uint32_t *__restrict__ SGl, float *__restrict__ M0l,
                                           float *__restrict__ M1l, LocT *__restrict__ LCl, size_t RSW, size_t RSL,
                                           uint32_t (&u)[4]) {
    using LO = LocOps<LocT>;
    const float INF = __int_as_float(0x7f800000);
    const uint32_t corr = (uint32_t)(d & 1) & (uint32_t)(!literal);  // (-1)^{d_i}, reading A1
    const float om0[4] = {R.m0.x, R.m0.y, R.m0.z, R.m0.w}, om1[4] = {R.m1.x, R.m1.y, R.m1.z, R.m1.w};
    float nm0[4] = {INF, INF, INF, INF}, nm1[4] = {INF, INF, INF, INF};
    int nloc[4] = {0, 0, 0, 0};
    uint32_t syn[4] = {0u, 0u, 0u, 0u}, wnew = 0;
#pragma unroll
    for (int p = 0; p < CH; p++) {
        if (p < d) {
            typename LO::W key{};
            if (!FIRST) key = LO::key(R.lc, p);
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const float sj = comp(R.sv[p], v);
                float x = sj;
                if (!FIRST) {
                    const float mag = LO::hit(key, v) ? om1[v] : om0[v];  // Obs. 1 (+ row parity)
                    x = sj - flip31(mag, R.wold << (31 - 4 * p - v));     // lambda_k - eta^prev_{i,k}
                }
                const float ax = fabsf(x);
                const bool lt = ax < nm0[v];  // first strict minimum (A13)
                nm1[v] = fminf(nm1[v], fmaxf(nm0[v], ax));
                nm0[v] = fminf(nm0[v], ax);
                nloc[v] = lt ? p : nloc[v];
                if (EARLY) syn[v] ^= __float_as_uint(sj) - 1u;      // bit 31: slice(s_j) == 0
                wnew |= (__float_as_uint(x) >> 31) << (4 * p + v);  // sign(0) = +1
            }
        }
    }
    SGl[(size_t)i * RSW] = wnew;
    // sign parity per frame (Obs. 2): XOR of bits v, v+4, ..., of the new sign word, times (-1)^{d_i}
    uint32_t pw = wnew ^ (wnew >> 16);
    pw ^= pw >> 8;
    pw ^= pw >> 4;
    pw ^= corr ? 0xfu : 0u;
    const uint32_t s0 = pw << 31, s1 = (pw << 30) & 0x80000000u, s2 = (pw << 29) & 0x80000000u,
                   s3 = (pw << 28) & 0x80000000u;
    st4(M0l + (size_t)i * RSW,
        make_float4(__uint_as_float(__float_as_uint(nm0[0]) | s0), __uint_as_float(__float_as_uint(nm0[1]) | s1),
                    __uint_as_float(__float_as_uint(nm0[2]) | s2), __uint_as_float(__float_as_uint(nm0[3]) | s3)));
    st4(M1l + (size_t)i * RSW,
        make_float4(__uint_as_float(__float_as_uint(nm1[0]) | s0), __uint_as_float(__float_as_uint(nm1[1]) | s1),
                    __uint_as_float(__float_as_uint(nm1[2]) | s2), __uint_as_float(__float_as_uint(nm1[3]) | s3)));
    LO::store(LCl + (size_t)i * RSL, nloc);
    if (EARLY) {
        const uint32_t dp = (uint32_t)(d & 1);  // XOR_j b_j = d_i mod 2 xor XOR_j (1 - b_j)
#pragma unroll
        for (int v = 0; v < 4; v++) u[v] |= __ballot_sync(FULL, ((syn[v] >> 31) ^ dp) != 0u);
    }
}

template <int CH, typename LocT, bool FIRST, bool EARLY, bool DB>
__global__ void __launch_bounds__(CN_T, (DB ? 2 : CN1_MINB) * CTA / CN_T)
    k_cn_pipe(Graph g, StreamState w, int k, int rows_per_cta, int literal, const int *kdev) {
    if (kdev) k = *kdev;  // body index supplied by the graph-driven loop
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t s_u[4];
    const int cnt = w.tcount[k & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) w.tcount[(k + 1) & 1] = 0;  // rebuilt by k_bn of body k
    if ((int)blockIdx.y >= cnt) return;  // active tiles are compacted to the front of the list
    const int t = w.tlist[(size_t)(k & 1) * w.T + blockIdx.y];
    if (EARLY) {
        if (threadIdx.x < 4) s_u[threadIdx.x] = 0;
        __syncthreads();
    }
    const int m = g.m, n = g.n;
    const float *__restrict__ Sl = w.s + (size_t)t * n * TILE + 4 * lane;
    // the tile's row records: [min0 512 B][min1 512 B][loc 128 x sizeof(LocT)][sign words 128 x wr]
    unsigned char *RB = w.rst + (size_t)t * m * w.rs;
    const size_t RSW = (size_t)w.rs / 4, RSL = (size_t)w.rs / sizeof(LocT);  // row strides
    float *__restrict__ M0l = reinterpret_cast<float *>(RB) + 4 * lane;
    float *__restrict__ M1l = reinterpret_cast<float *>(RB) + 128 + 4 * lane;
    LocT *__restrict__ LCl = reinterpret_cast<LocT *>(RB + 1024) + 4 * lane;
    uint32_t *__restrict__ SGl = reinterpret_cast<uint32_t *>(RB + 1024 + 128 * sizeof(LocT)) + lane;
    const int i0 = blockIdx.x * rows_per_cta + warp, i1 = min(m, blockIdx.x * rows_per_cta + rows_per_cta);
    constexpr int NW = CN_T / 32;  // warps per CTA
    const int nr = i0 < i1 ? (i1 - i0 + NW - 1) / NW : 0;  // rows of this warp (<= 32)
    uint32_t u[4] = {0u, 0u, 0u, 0u};
    // a warp without rows must still reach the CTA barrier of the EARLY epilogue
    if (nr > 0) {
    int ra = 0, rb = 0;  // lane q: row_ptr of the warp's row q
    if (lane < nr) {
        ra = __ldg(g.row_ptr + i0 + NW * lane);
        rb = __ldg(g.row_ptr + i0 + NW * lane + 1);
    }
    auto row_of = [&](int q) { return i0 + NW * min(q, nr - 1); };
    auto deg_of = [&](int q) { return __shfl_sync(FULL, rb, q & 31) - __shfl_sync(FULL, ra, q & 31); };
    auto cols_of = [&](int q) {  // lane p: column of edge p of row q (0 past the degree / past the rows)
        const int a = __shfl_sync(FULL, ra, q & 31), d = __shfl_sync(FULL, rb, q & 31) - a;
        return (q < nr && lane < d) ? __ldg(g.col_idx + a + lane) : 0;
    };
    if (!DB) {  // one row buffer: all loads of a row in flight together, more warps per SM
        CnRow<CH, LocT> A;
        int cj = cols_of(0);
        for (int q = 0; q < nr; q++) {
            cn_fetch<CH, LocT, FIRST>(A, cj, row_of(q), Sl, SGl, M0l, M1l, LCl, RSW, RSL);
            cj = cols_of(q + 1);
            cn_compute<CH, LocT, FIRST, EARLY>(A, row_of(q), deg_of(q), literal, SGl, M0l, M1l, LCl, RSW, RSL, u);
        }
    } else {
    CnRow<CH, LocT> A, B;
    int cjA = cols_of(0), cjB = cols_of(1);
    cn_fetch<CH, LocT, FIRST>(A, cjA, row_of(0), Sl, SGl, M0l, M1l, LCl, RSW, RSL);
    cjA = cols_of(2);
    for (int q = 0; q < nr; q += 2) {
        cn_fetch<CH, LocT, FIRST>(B, cjB, row_of(q + 1), Sl, SGl, M0l, M1l, LCl, RSW, RSL);
        cjB = cols_of(q + 3);
        cn_compute<CH, LocT, FIRST, EARLY>(A, row_of(q), deg_of(q), literal, SGl, M0l, M1l, LCl, RSW, RSL, u);
        if (q + 1 >= nr) break;
        cn_fetch<CH, LocT, FIRST>(A, cjA, row_of(q + 2), Sl, SGl, M0l, M1l, LCl, RSW, RSL);
        cjA = cols_of(q + 4);
        cn_compute<CH, LocT, FIRST, EARLY>(B, row_of(q + 1), deg_of(q + 1), literal, SGl, M0l, M1l, LCl, RSW, RSL, u);
    }
    }
    }  // nr > 0
    if (EARLY) {
        if (lane == 0) {
#pragma unroll
            for (int v = 0; v < 4; v++)
                if (u[v]) atomicOr(&s_u[v], u[v]);
        }
        __syncthreads();
        if (threadIdx.x < 4 && s_u[threadIdx.x])
            atomicOr(w.unsat + ((size_t)(k & 1) * w.T + t) * 4 + threadIdx.x, s_u[threadIdx.x]);
    }
}

// ------------------------------------------------------------------------------------------------
// a5/a6: bit-node sweep of loop body k; stops frames whose b^(k-1) satisfied every check.
// One edge at a time with few registers and many warps (6 CTAs per SM): the loads of an edge depend
// only on its broadcast record, and the warps of the SM keep enough of them in flight.
// ------------------------------------------------------------------------------------------------
template <typename LocT, bool EARLY>
__global__ void __launch_bounds__(BNL_T, BNL_MINB * CTA / BNL_T)
    k_bn(Graph g, StreamState w, int k, int cols_per_cta, int literal, const int *kdev, int check_every) {
    using LO = LocOps<LocT>;
    if (kdev) k = *kdev;
    (void)literal;
    const int lane = threadIdx.x & 31;
    const int T = w.T;
    const int cnt = w.tcount[k & 1];
    if ((int)blockIdx.y >= cnt) return;
    const int t = w.tlist[(size_t)(k & 1) * T + blockIdx.y];
    const int cblk = blockIdx.x;
    uint4 act = make_uint4(FULL, FULL, FULL, FULL);
    if (EARLY) {
        // the syndrome of k_cn(k) tests b^(k-1); it may stop frames only at a check point (k-1) % T == 0
        const bool check = ((k - 1) % check_every) == 0;
        const uint4 ua = check ? ldu4(w.unsat + ((size_t)(k & 1) * T + t) * 4) : make_uint4(FULL, FULL, FULL, FULL);
        const uint4 dw = ldu4(w.done + (size_t)t * 4);
        const uint4 newly = make_uint4(~ua.x & ~dw.x, ~ua.y & ~dw.y, ~ua.z & ~dw.z, ~ua.w & ~dw.w);
        act = make_uint4(ua.x & ~dw.x, ua.y & ~dw.y, ua.z & ~dw.z, ua.w & ~dw.w);
        // every thread must read `done` before the tile's bookkeeping item rewrites it (other items of
        // the tile may see either value: act is the same for both, since newly and ua are disjoint)
        __syncthreads();
        if (cblk == 0) {
            const int tid = threadIdx.x;
            if (tid < 4) {
                w.done[(size_t)t * 4 + tid] = comp(dw, tid) | comp(newly, tid);
                w.unsat[((size_t)((k + 1) & 1) * T + t) * 4 + tid] = 0;  // buffer of body k+1
            }
            if (tid < TILE && ((comp(newly, tid & 3) >> (tid >> 2)) & 1u))
                w.iters[(size_t)t * TILE + tid] = k - 1;  // stopped after k-1 bodies
            if (tid == 0 && (act.x | act.y | act.z | act.w)) {  // tile still runs in body k+1
                const int pos = atomicAdd(w.tcount + ((k + 1) & 1), 1);
                w.tlist[(size_t)((k + 1) & 1) * T + pos] = t;
            }
        }
        if ((act.x | act.y | act.z | act.w) == 0) return;
    } else if (cblk == 0 && threadIdx.x == 0) {
        const int pos = atomicAdd(w.tcount + ((k + 1) & 1), 1);
        w.tlist[(size_t)((k + 1) & 1) * T + pos] = t;
    }
    const unsigned mine = ((act.x >> lane) & 1u) | (((act.y >> lane) & 1u) << 1) | (((act.z >> lane) & 1u) << 2) |
                          (((act.w >> lane) & 1u) << 3);
    const int m = g.m, n = g.n, wr = g.wr;
    // the tile's row records: [min0 512 B][min1 512 B][loc 128 x sizeof(LocT)][sign words 128 x wr]
    unsigned char *RB = w.rst + (size_t)t * m * w.rs;
    const size_t RSW = (size_t)w.rs / 4, RSL = (size_t)w.rs / sizeof(LocT);  // row strides
    const float *__restrict__ M0l = reinterpret_cast<float *>(RB) + 4 * lane;
    const float *__restrict__ M1l = reinterpret_cast<float *>(RB) + 128 + 4 * lane;
    const LocT *__restrict__ LCl = reinterpret_cast<LocT *>(RB + 1024) + 4 * lane;
    const uint32_t *__restrict__ SGl = reinterpret_cast<uint32_t *>(RB + 1024 + 128 * sizeof(LocT)) + lane;
    const float *__restrict__ Rl = w.r + (size_t)t * n * TILE + 4 * lane;
    float *__restrict__ Sl = w.s + (size_t)t * n * TILE + 4 * lane;
    const int warp = threadIdx.x >> 5;
    const int j1 = min(n, cblk * cols_per_cta + cols_per_cta);
    // one edge at a time, few registers, many warps (6 CTAs per SM): the loads of an edge depend only
    // on its (broadcast) record, and the warps of the SM keep enough of them in flight
    for (int j = cblk * cols_per_cta + warp; j < j1; j += BNL_T / 32) {
        const int c0 = __ldg(g.col_ptr + j), dv = __ldg(g.col_ptr + j + 1) - c0;
        const float4 rv = ld4(Rl + (size_t)j * TILE);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int q = 0; q < dv; q++) {
            const int4 ed = __ldg(g.bn_edge + c0 + q);  // {e, i, p, -}, ascending i
            const size_t ro = (size_t)ed.y * RSW;  // row record of row i
            const float4 m0 = ld4(M0l + ro), m1 = ld4(M1l + ro);
            const typename LO::W key = LO::key(LO::load(LCl + (size_t)ed.y * RSL), ed.z);
            const uint32_t ws = SGl[ro + (ed.z >> 3) * 32] << (28 - 4 * (ed.z & 7));
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const float mag = LO::hit(key, v) ? comp(m1, v) : comp(m0, v);  // Obs. 1
                acc[v] = acc[v] + flip31(mag, ws << (3 - v));                   // ascending rows from +0.0 (A14)
            }
        }
        float *o = Sl + (size_t)j * TILE;
        if (mine == 0xFu) {
            st4(o, make_float4(acc[0] + rv.x, acc[1] + rv.y, acc[2] + rv.z, acc[3] + rv.w));
        } else if (mine) {  // frozen frames keep their s
            if (mine & 1u) o[0] = acc[0] + rv.x;
            if (mine & 2u) o[1] = acc[1] + rv.y;
            if (mine & 4u) o[2] = acc[2] + rv.z;
            if (mine & 8u) o[3] = acc[3] + rv.w;
        }
    }
}

// ------------------------------------------------------------------------------------------------
// a6: syndrome of b^(L) (the test after the last body), into unsat[slot].
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(CTA) k_syndrome(Graph g, StreamState w, int slot, int rows_per_cta) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t s_u[4];
    const int cnt = w.tcount[slot];  // tiles still running after the last body
    if ((int)blockIdx.y >= cnt) return;
    {
    const int t = w.tlist[(size_t)slot * w.T + blockIdx.y];
    const int rblk = blockIdx.x;
    if (threadIdx.x < 4) s_u[threadIdx.x] = 0;
    __syncthreads();
    const size_t tn = (size_t)t * g.n;
    const int i0 = rblk * rows_per_cta, i1 = min(g.m, i0 + rows_per_cta);
    uint32_t u[4] = {0, 0, 0, 0};
    for (int i = i0 + warp; i < i1; i += CTA / 32) {
        const int a = __ldg(g.row_ptr + i), d = __ldg(g.row_ptr + i + 1) - a;
        unsigned syn = 0;
        for (int p = 0; p < d; p++) {
            const int j = __ldg(g.col_idx + a + p);
            const float4 sv = ld4(w.s + (tn + j) * TILE + 4 * lane);
            syn ^= (unsigned)(sv.x > 0.f) | ((unsigned)(sv.y > 0.f) << 1) | ((unsigned)(sv.z > 0.f) << 2) |
                   ((unsigned)(sv.w > 0.f) << 3);
        }
#pragma unroll
        for (int v = 0; v < 4; v++) u[v] |= __ballot_sync(FULL, (syn >> v) & 1u);
    }
    if (lane == 0)
#pragma unroll
        for (int v = 0; v < 4; v++)
            if (u[v]) atomicOr(&s_u[v], u[v]);
    __syncthreads();
    if (threadIdx.x < 4 && s_u[threadIdx.x])
        atomicOr(w.unsat + ((size_t)slot * w.T + t) * 4 + threadIdx.x, s_u[threadIdx.x]);
    }
}

// ------------------------------------------------------------------------------------------------
// a7: stage-out.  s [T][n][128] -> posterior [F][n], bits = slice(s) [F][n]; per-frame counters.
// ------------------------------------------------------------------------------------------------
constexpr int FIN_SUB = 8;  // 32-column sub-blocks per finalize CTA

__global__ void __launch_bounds__(CTA) k_finalize(StreamState w, int n, int64_t frames, float *__restrict__ post,
                                                  uint8_t *__restrict__ bits) {
    __shared__ float ts[32][TILE + 1];
    __shared__ float tr[32][TILE + 1];
    const int t = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // per-frame counters over the CTA's 256 columns: lane q holds frame warp + 8q (q < 16); one atomic
    // per frame and CTA instead of one per 32 columns
    int be_acc = 0, raw_acc = 0;
    bool nz_acc = false;
    for (int sb = 0; sb < FIN_SUB; sb++) {
        const int j0 = (blockIdx.x * FIN_SUB + sb) * 32;
        if (j0 >= n) break;
        for (int jl = warp; jl < 32; jl += CTA / 32) {
            const int j = j0 + jl;
            if (j >= n) break;
            const size_t base = ((size_t)t * n + j) * TILE;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                ts[jl][lane + 32 * q] = w.s[base + lane + 32 * q];
                tr[jl][lane + 32 * q] = w.r[base + lane + 32 * q];
            }
        }
        __syncthreads();
        const int j = j0 + lane;
        const bool jv = j < n;
#pragma unroll 4
        for (int q = 0; q < TILE / (CTA / 32); q++) {
            const int fl = warp + (CTA / 32) * q;
            const int64_t f = (int64_t)t * TILE + fl;
            if (f >= frames) break;
            const float sv = ts[lane][fl];
            const bool b = jv && sv > 0.f;  // Eq. slice
            if (jv) {
                if (post) post[f * n + j] = sv;
                if (bits) bits[f * n + j] = (uint8_t)b;
            }
            const int be = __popc(__ballot_sync(FULL, b));
            const int raw = __popc(__ballot_sync(FULL, jv && tr[lane][fl] > 0.f));
            const bool nz = __any_sync(FULL, jv && fabsf(sv) <= 1e-4f);
            if (lane == q) {
                be_acc += be;
                raw_acc += raw;
                nz_acc = nz_acc || nz;
            }
        }
        __syncthreads();  // the next sub-block overwrites ts / tr
    }
    if (lane < TILE / (CTA / 32)) {
        const int fl = warp + (CTA / 32) * lane;
        if ((int64_t)t * TILE + fl < frames) {
            if (be_acc) atomicAdd(w.fbe + (size_t)t * TILE + fl, be_acc);
            if (raw_acc) atomicAdd(w.fraw + (size_t)t * TILE + fl, raw_acc);
            if (nz_acc) w.fnz[(size_t)t * TILE + fl] = 1;
        }
    }
}

// per-frame k, isCodeword and the 8 accumulated counters
__global__ void __launch_bounds__(CTA) k_frame_stats(StreamState w, int64_t frames, int L, int early, int slot,
                                                     int32_t *__restrict__ iters_out, uint8_t *__restrict__ conv_out,
                                                     unsigned long long *__restrict__ stats) {
    __shared__ unsigned long long s_acc[8];
    if (threadIdx.x < 8) s_acc[threadIdx.x] = 0;
    __syncthreads();
    const int64_t f = blockIdx.x * (int64_t)CTA + threadIdx.x;
    unsigned long long c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (f < frames) {
        const int64_t t = f / TILE;
        const int fl = (int)(f % TILE), ln = fl >> 2, v = fl & 3;
        int it = L, conv;
        const bool stopped = early && ((w.done[t * 4 + v] >> ln) & 1u);
        if (stopped) {
            it = w.iters[f];
            conv = 1;
        } else {
            conv = !((w.unsat[((int64_t)slot * w.T + t) * 4 + v] >> ln) & 1u);
        }
        if (iters_out) iters_out[f] = it;
        if (conv_out) conv_out[f] = (uint8_t)conv;
        const int be = w.fbe[f];
        c[0] = 1;
        c[1] = (unsigned long long)be;
        c[2] = be > 0;
        c[3] = (be > 0) && conv;
        c[4] = (unsigned long long)it;
        c[5] = conv;
        c[6] = w.fnz[f] != 0;
        c[7] = (unsigned long long)w.fraw[f];
    }
    if (stats) {
#pragma unroll
        for (int q = 0; q < 8; q++) {
            unsigned long long x = c[q];
            for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
            if ((threadIdx.x & 31) == 0 && x) atomicAdd(&s_acc[q], x);
        }
        __syncthreads();
        if (threadIdx.x < 8 && s_acc[threadIdx.x]) atomicAdd(stats + threadIdx.x, s_acc[threadIdx.x]);
    }
}

// Graph-driven loop control (CUDA conditional WHILE node): body k runs while k <= L and some tile
// still has a running frame.  On an early end, the list the final syndrome pass reads is emptied.
__global__ void k_loop_pre(StreamState w, int L, cudaGraphConditionalHandle h) {
    const int k = 2;
    const bool run = k <= L && w.tcount[k & 1] > 0;
    *w.kdev = k;
    if (run && w.nlaunch) *w.nlaunch += 3;  // check node, bit node, step of body k
    if (!run) w.tcount[(L + 1) & 1] = 0;
    cudaGraphSetConditional(h, run ? 1u : 0u);
}

__global__ void k_loop_step(StreamState w, int L, cudaGraphConditionalHandle h) {
    const int k = *w.kdev + 1;
    const bool run = k <= L && w.tcount[k & 1] > 0;
    *w.kdev = k;
    if (run && w.nlaunch) *w.nlaunch += 3;
    if (!run && k <= L) w.tcount[(L + 1) & 1] = 0;
    cudaGraphSetConditional(h, run ? 1u : 0u);
}

inline dim3 grid2(int64_t x, int y) { return dim3((unsigned)std::max<int64_t>(1, x), (unsigned)y); }

}  // namespace

int launch_stage_in(const Graph &g, const StreamState &w, const float *llr, int64_t frames, cudaStream_t st) {
    k_stage_in<<<grid2((g.n + 31) / 32, w.T), CTA, 0, st>>>(llr, frames, g.n, w.T, w.r, w.s, w.unsat, w.done, w.fbe,
                                                           w.fraw, w.fnz, w.tcount, w.tlist);
    return 1;
}

template <typename LT, bool F, bool EA>
void cn_launch(dim3 grid, cudaStream_t st, const Graph &g, const StreamState &w, int k, int rpc, int lit, int u,
               const int *kdev) {
    // u: 0 = single row buffer (default), 2 = two row buffers, 1 = generic kernel
    if (u != 1 && u != 2 && g.dmax <= 8) {
        if (g.dmax <= 4) k_cn_pipe<4, LT, F, EA, false><<<grid, CN_T, 0, st>>>(g, w, k, rpc, lit, kdev);
        else if (g.dmax <= 6) k_cn_pipe<6, LT, F, EA, false><<<grid, CN_T, 0, st>>>(g, w, k, rpc, lit, kdev);
        else if (g.dmax == 7) k_cn_pipe<7, LT, F, EA, false><<<grid, CN_T, 0, st>>>(g, w, k, rpc, lit, kdev);
        else k_cn_pipe<8, LT, F, EA, false><<<grid, CN_T, 0, st>>>(g, w, k, rpc, lit, kdev);
    } else if (u == 2 && g.dmax <= 6) k_cn_pipe<6, LT, F, EA, true><<<grid, CN_T, 0, st>>>(g, w, k, rpc, lit, kdev);
    else if (u == 2 && g.dmax <= 8) k_cn_pipe<8, LT, F, EA, true><<<grid, CN_T, 0, st>>>(g, w, k, rpc, lit, kdev);
    else k_cn<LT, F, EA><<<grid, CTA, 0, st>>>(g, w, k, rpc, lit, kdev);
}

template <typename LT, bool EA>
void bn_launch(dim3 grid, cudaStream_t st, const Graph &g, const StreamState &w, int k, int cpc, int lit, int u,
               const int *kdev, int te) {
    (void)grid;
    (void)cpc;
    (void)u;
    k_bn<LT, EA><<<grid2((g.n + BNL_COLS - 1) / BNL_COLS, w.T), BNL_T, 0, st>>>(g, w, k, BNL_COLS, lit, kdev, te);
}

int launch_check_node(const Graph &g, const StreamState &w, int k, bool first, bool early, bool literal, bool loc16,
                      const StreamLaunch &cfg, cudaStream_t st, const int *kdev) {
    const dim3 grid = grid2((g.m + cfg.rows_per_cta - 1) / cfg.rows_per_cta, w.T);
    const int lit = literal ? 1 : 0, rpc = cfg.rows_per_cta, u = cfg.cn_unroll;
    if (loc16) {
        if (first) { if (early) cn_launch<uint16_t, true, true>(grid, st, g, w, k, rpc, lit, u, kdev);
                     else cn_launch<uint16_t, true, false>(grid, st, g, w, k, rpc, lit, u, kdev); }
        else { if (early) cn_launch<uint16_t, false, true>(grid, st, g, w, k, rpc, lit, u, kdev);
               else cn_launch<uint16_t, false, false>(grid, st, g, w, k, rpc, lit, u, kdev); }
    } else {
        if (first) { if (early) cn_launch<uint8_t, true, true>(grid, st, g, w, k, rpc, lit, u, kdev);
                     else cn_launch<uint8_t, true, false>(grid, st, g, w, k, rpc, lit, u, kdev); }
        else { if (early) cn_launch<uint8_t, false, true>(grid, st, g, w, k, rpc, lit, u, kdev);
               else cn_launch<uint8_t, false, false>(grid, st, g, w, k, rpc, lit, u, kdev); }
    }
    return 1;
}

int launch_bit_node(const Graph &g, const StreamState &w, int k, bool early, bool literal, bool loc16,
                    const StreamLaunch &cfg, cudaStream_t st, const int *kdev) {
    const dim3 grid = grid2((g.n + BNL_COLS - 1) / BNL_COLS, w.T);
    const int lit = literal ? 1 : 0, cpc = BNL_COLS, u = 0;
    if (loc16) {
        if (early) bn_launch<uint16_t, true>(grid, st, g, w, k, cpc, lit, u, kdev, cfg.check_every);
        else bn_launch<uint16_t, false>(grid, st, g, w, k, cpc, lit, u, kdev, cfg.check_every);
    } else {
        if (early) bn_launch<uint8_t, true>(grid, st, g, w, k, cpc, lit, u, kdev, cfg.check_every);
        else bn_launch<uint8_t, false>(grid, st, g, w, k, cpc, lit, u, kdev, cfg.check_every);
    }
    return 1;
}

int launch_syndrome(const Graph &g, const StreamState &w, int slot, const StreamLaunch &cfg, cudaStream_t st) {
    k_syndrome<<<grid2((g.m + cfg.rows_per_cta - 1) / cfg.rows_per_cta, w.T), CTA, 0, st>>>(g, w, slot,
                                                                                             cfg.rows_per_cta);
    return 1;
}

int launch_loop_pre(const StreamState &w, int L, cudaGraphConditionalHandle h, cudaStream_t st) {
    k_loop_pre<<<1, 1, 0, st>>>(w, L, h);
    return 1;
}

int launch_loop_step(const StreamState &w, int L, cudaGraphConditionalHandle h, cudaStream_t st) {
    k_loop_step<<<1, 1, 0, st>>>(w, L, h);
    return 1;
}

int launch_finalize(const Graph &g, const StreamState &w, int64_t frames, float *posterior, uint8_t *bits,
                    cudaStream_t st) {
    k_finalize<<<grid2((g.n + 32 * FIN_SUB - 1) / (32 * FIN_SUB), w.T), CTA, 0, st>>>(w, g.n, frames, posterior, bits);
    return 1;
}

int launch_frame_stats(const Graph &g, const StreamState &w, int64_t frames, int L, bool early, int final_slot,
                       int32_t *iters_out, uint8_t *conv_out, unsigned long long *stats, cudaStream_t st) {
    (void)g;
    k_frame_stats<<<(unsigned)std::max<int64_t>(1, (frames + CTA - 1) / CTA), CTA, 0, st>>>(
        w, frames, L, early ? 1 : 0, final_slot, iters_out, conv_out, stats);
    return 1;
}

}  // namespace ldpc
