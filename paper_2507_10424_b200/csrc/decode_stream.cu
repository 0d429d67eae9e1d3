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

__device__ __forceinline__ float4 ldg4(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }
__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ void st4(float *p, float4 v) { *reinterpret_cast<float4 *>(p) = v; }
__device__ __forceinline__ uint4 ldu4(const uint32_t *p) { return *reinterpret_cast<const uint4 *>(p); }

// ------------------------------------------------------------------------------------------------
// a2: stage-in.  llr [F][n] -> r, s [T][n][128] (s = r), init per-tile flags.
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
            s[base + lane + 32 * q] = v;
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
// a3/a4/a6: check-node sweep of loop body k (k = 1..L), fused syndrome of b^(k-1).
// FIRST: eta^prev = 0, so no old state is read.
// Sign words: per (tile, edge) four u32; lane l's four bits (frames 4l..4l+3) are the nibble at bits
// 4*(l%8) of word l/8, so a lane reads one u32 per edge.  The row parity stored in min0's sign bit
// already includes the (-1)^{d_i} factor of reading A1.
// The edges of a row are processed in chunks of CN_U: all index, s and sign loads of a chunk are
// issued before any arithmetic, so each warp keeps 2*CN_U loads in flight.
// ------------------------------------------------------------------------------------------------
template <int U>
struct MinBlocks {
    static constexpr int value = U <= 1 ? 4 : U == 2 ? 3 : 2;  // register budget 64 / 85 / 128 per thread
};

template <typename LocT, bool FIRST, bool EARLY, int CN_U>
__global__ void __launch_bounds__(CTA, MinBlocks<CN_U>::value)
    k_cn(Graph g, StreamState w, int k, int rows_per_cta, int literal, const int *kdev) {
    using L4 = typename Vec4<LocT>::type;
    if (kdev) k = *kdev;  // body index supplied by the graph-driven loop
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t s_u[4];
    // the tiles of body k are the ones with a running frame (list rebuilt by k_bn of body k-1)
    const int cnt = w.tcount[k & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) w.tcount[(k + 1) & 1] = 0;  // rebuilt by k_bn of body k
    if ((int)blockIdx.y >= cnt) return;  // active tiles are compacted to the front of the list
    {
    const int t = w.tlist[(size_t)(k & 1) * w.T + blockIdx.y];
    const int rblk = blockIdx.x;
    if (EARLY) {
        if (threadIdx.x < 4) s_u[threadIdx.x] = 0;
        __syncthreads();
    }
    const int *__restrict__ row_ptr = g.row_ptr;
    const int *__restrict__ col_idx = g.col_idx;
    const float *__restrict__ S = w.s;
    uint32_t *__restrict__ SG = w.sgn;
    float *__restrict__ M0 = w.min0;
    float *__restrict__ M1 = w.min1;
    LocT *__restrict__ LC = reinterpret_cast<LocT *>(w.loc);
    const int m = g.m, n = g.n, E = g.E;
    const size_t tm = (size_t)t * m, tn = (size_t)t * n, tE = (size_t)t * E;
    const int sh = 4 * (lane & 7), wsel = lane >> 3;
    const int i0 = rblk * rows_per_cta, i1 = min(m, i0 + rows_per_cta);
    uint32_t u0 = 0, u1 = 0, u2 = 0, u3 = 0;
    for (int i = i0 + warp; i < i1; i += CTA / 32) {
        const int a = __ldg(row_ptr + i), d = __ldg(row_ptr + i + 1) - a;
        const unsigned corr = (unsigned)(d & 1) & (unsigned)(!literal);  // (-1)^{d_i}, reading A1
        const size_t st = (tm + i) * TILE + 4 * lane;
        float4 om0 = make_float4(0.f, 0.f, 0.f, 0.f), om1 = om0;
        L4 olc{};
        if (!FIRST) {
            om0 = ld4(M0 + st);
            om1 = ld4(M1 + st);
            olc = *reinterpret_cast<const L4 *>(LC + st);
        }
        float nm0[4], nm1[4];
        int nloc[4];
        unsigned npar = 0, syn = 0;
#pragma unroll
        for (int v = 0; v < 4; v++) {
            nm0[v] = __int_as_float(0x7f800000);
            nm1[v] = __int_as_float(0x7f800000);
            nloc[v] = 0;
        }
        for (int p0 = 0; p0 < d; p0 += CN_U) {
            int jj[CN_U];
            float4 sv[CN_U];
            unsigned sw[CN_U];
#pragma unroll
            for (int u = 0; u < CN_U; u++) jj[u] = (p0 + u < d) ? __ldg(col_idx + a + p0 + u) : 0;
#pragma unroll
            for (int u = 0; u < CN_U; u++) {
                if (p0 + u < d) {
                    sv[u] = ld4(S + (tn + jj[u]) * TILE + 4 * lane);
                    sw[u] = FIRST ? 0u : (SG[(tE + a + p0 + u) * 4 + wsel] >> sh);
                }
            }
#pragma unroll
            for (int u = 0; u < CN_U; u++) {
                if (p0 + u >= d) break;
                const int p = p0 + u;
                unsigned nib = 0;
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    const float sj = comp(sv[u], v);
                    float x = sj;
                    if (!FIRST) {
                        const float m0v = comp(om0, v);
                        const float mag = (p == compl4(olc, v)) ? comp(om1, v) : fabsf(m0v);  // Obs. 1
                        const unsigned neg_eta = ((sw[u] >> v) & 1u) ^ (__float_as_uint(m0v) >> 31);  // Obs. 2
                        x = sj - (neg_eta ? -mag : mag);  // lambda_k - eta^prev_{i,k}
                    }
                    const float ax = fabsf(x);
                    const bool lt = ax < nm0[v];  // first strict minimum (A13)
                    nm1[v] = fminf(nm1[v], fmaxf(nm0[v], ax));
                    nm0[v] = fminf(nm0[v], ax);
                    nloc[v] = lt ? p : nloc[v];
                    nib |= (unsigned)(x < 0.f) << v;  // sign(0) = +1
                    if (EARLY) syn ^= (unsigned)(sj > 0.f) << v;  // b_j = slice(s_j)
                }
                npar ^= nib;
                unsigned word = nib << sh;
                word |= __shfl_xor_sync(FULL, word, 1);
                word |= __shfl_xor_sync(FULL, word, 2);
                word |= __shfl_xor_sync(FULL, word, 4);
                if ((lane & 7) == 0) SG[(tE + a + p) * 4 + wsel] = word;
            }
        }
        const unsigned pc = npar ^ (corr ? 0xfu : 0u);
        float4 o0;
        o0.x = __uint_as_float(__float_as_uint(nm0[0]) | ((pc & 1u) << 31));
        o0.y = __uint_as_float(__float_as_uint(nm0[1]) | (((pc >> 1) & 1u) << 31));
        o0.z = __uint_as_float(__float_as_uint(nm0[2]) | (((pc >> 2) & 1u) << 31));
        o0.w = __uint_as_float(__float_as_uint(nm0[3]) | (((pc >> 3) & 1u) << 31));
        st4(M0 + st, o0);
        st4(M1 + st, make_float4(nm1[0], nm1[1], nm1[2], nm1[3]));
        L4 nl;
        nl.x = (LocT)nloc[0];
        nl.y = (LocT)nloc[1];
        nl.z = (LocT)nloc[2];
        nl.w = (LocT)nloc[3];
        *reinterpret_cast<L4 *>(LC + st) = nl;
        if (EARLY) {
            u0 |= __ballot_sync(FULL, syn & 1u);
            u1 |= __ballot_sync(FULL, syn & 2u);
            u2 |= __ballot_sync(FULL, syn & 4u);
            u3 |= __ballot_sync(FULL, syn & 8u);
        }
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
}

// ------------------------------------------------------------------------------------------------
// Check-node sweep with TMA-style bulk-copy staging (cp.async.bulk + mbarrier, per-warp double
// buffer).  A warp owns ROWS_PER_WARP rows of the block; while it computes row q from shared
// memory, the bulk copies of row q+2 (the d gathered 512-byte s segments, the d sign words and the
// old row state) are in flight, so every warp keeps a whole row of loads outstanding without
// holding them in registers.  Same arithmetic and results as k_cn.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

constexpr int ROWS_PER_WARP = 8;

// shared-memory bytes of one staging buffer for rows of degree <= dm
__host__ __device__ constexpr int cn_stage_bytes(int dm, int locb) { return dm * 512 + dm * 16 + 1024 + 128 * locb + 16; }

template <typename LocT, bool FIRST, bool EARLY>
__global__ void __launch_bounds__(CTA) k_cn_tma(Graph g, StreamState w, int k, int dm, int literal, const int *kdev) {
    using L4 = typename Vec4<LocT>::type;
    if (kdev) k = *kdev;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint32_t s_u[4];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cnt = w.tcount[k & 1];
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) w.tcount[(k + 1) & 1] = 0;
    if ((int)blockIdx.y >= cnt) return;  // active tiles are compacted to the front of the list
    const int t = w.tlist[(size_t)(k & 1) * w.T + blockIdx.y];
    if (EARLY && threadIdx.x < 4) s_u[threadIdx.x] = 0;
    const int sbytes = cn_stage_bytes(dm, (int)sizeof(LocT));
    unsigned char *wbase = smem + (size_t)warp * 2 * sbytes;
    // stage layout: s[dm][128] f32 | sw[dm][4] u32 | min0[128] | min1[128] | loc[128] | mbarrier
    auto sbuf = [&](int b) { return reinterpret_cast<float *>(wbase + b * sbytes); };
    auto swbuf = [&](int b) { return reinterpret_cast<uint32_t *>(wbase + b * sbytes + dm * 512); };
    auto m0buf = [&](int b) { return reinterpret_cast<float *>(wbase + b * sbytes + dm * 528); };
    auto m1buf = [&](int b) { return reinterpret_cast<float *>(wbase + b * sbytes + dm * 528 + 512); };
    auto lcbuf = [&](int b) { return reinterpret_cast<LocT *>(wbase + b * sbytes + dm * 528 + 1024); };
    auto bar = [&](int b) {
        return reinterpret_cast<uint64_t *>(wbase + b * sbytes + dm * 528 + 1024 + 128 * sizeof(LocT));
    };
    if (lane == 0) {
        mbar_init(bar(0), 1);
        mbar_init(bar(1), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int *__restrict__ row_ptr = g.row_ptr;
    const int *__restrict__ col_idx = g.col_idx;
    const float *S = w.s;
    uint32_t *SG = w.sgn;
    float *M0 = w.min0;
    float *M1 = w.min1;
    LocT *LC = reinterpret_cast<LocT *>(w.loc);
    const int m = g.m, n = g.n, E = g.E;
    const size_t tm = (size_t)t * m, tn = (size_t)t * n, tE = (size_t)t * E;
    const int sh = 4 * (lane & 7), wsel = lane >> 3;
    const int rpc = (CTA / 32) * ROWS_PER_WARP;
    const int i0 = blockIdx.x * rpc;
    const int nq = max(0, min(ROWS_PER_WARP, (m - i0 - warp + (CTA / 32) - 1) / (CTA / 32)));

    auto stage = [&](int q, int b) {
        const int i = i0 + warp + (CTA / 32) * q;
        const int a = __ldg(row_ptr + i), d = __ldg(row_ptr + i + 1) - a;
        const unsigned bytes = (unsigned)d * (FIRST ? 512u : 528u) + (FIRST ? 0u : (unsigned)(1024 + 128 * sizeof(LocT)));
        if (lane == 0) mbar_expect_tx(bar(b), bytes);
        __syncwarp();
        for (int p = lane; p < d; p += 32) {
            const int j = __ldg(col_idx + a + p);
            bulk_g2s(sbuf(b) + p * TILE, S + (tn + j) * TILE, 512, bar(b));
            if (!FIRST) bulk_g2s(swbuf(b) + p * 4, SG + (tE + a + p) * 4, 16, bar(b));
        }
        if (!FIRST && lane == 31) {
            const size_t st = (tm + i) * TILE;
            bulk_g2s(m0buf(b), M0 + st, 512, bar(b));
            bulk_g2s(m1buf(b), M1 + st, 512, bar(b));
            bulk_g2s(lcbuf(b), LC + st, 128 * sizeof(LocT), bar(b));
        }
    };

    if (nq > 0) stage(0, 0);
    if (nq > 1) stage(1, 1);
    uint32_t u0 = 0, u1 = 0, u2 = 0, u3 = 0;
    for (int q = 0; q < nq; q++) {
        const int b = q & 1;
        const int i = i0 + warp + (CTA / 32) * q;
        const int a = __ldg(row_ptr + i), d = __ldg(row_ptr + i + 1) - a;
        const unsigned corr = (unsigned)(d & 1) & (unsigned)(!literal);  // (-1)^{d_i}, reading A1
        mbar_wait(bar(b), (unsigned)(q >> 1) & 1u);
        float4 om0 = make_float4(0.f, 0.f, 0.f, 0.f), om1 = om0;
        L4 olc{};
        if (!FIRST) {
            om0 = *reinterpret_cast<const float4 *>(m0buf(b) + 4 * lane);
            om1 = *reinterpret_cast<const float4 *>(m1buf(b) + 4 * lane);
            olc = *reinterpret_cast<const L4 *>(lcbuf(b) + 4 * lane);
        }
        float nm0[4], nm1[4];
        int nloc[4];
        unsigned npar = 0, syn = 0;
#pragma unroll
        for (int v = 0; v < 4; v++) {
            nm0[v] = __int_as_float(0x7f800000);
            nm1[v] = __int_as_float(0x7f800000);
            nloc[v] = 0;
        }
        for (int p = 0; p < d; p++) {
            const float4 sv = *reinterpret_cast<const float4 *>(sbuf(b) + p * TILE + 4 * lane);
            const unsigned sw = FIRST ? 0u : (swbuf(b)[p * 4 + wsel] >> sh);
            unsigned nib = 0;
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const float sj = comp(sv, v);
                float x = sj;
                if (!FIRST) {
                    const float m0v = comp(om0, v);
                    const float mag = (p == compl4(olc, v)) ? comp(om1, v) : fabsf(m0v);  // Obs. 1
                    const unsigned neg_eta = ((sw >> v) & 1u) ^ (__float_as_uint(m0v) >> 31);  // Obs. 2
                    x = sj - (neg_eta ? -mag : mag);  // lambda_k - eta^prev_{i,k}
                }
                const float ax = fabsf(x);
                const bool lt = ax < nm0[v];  // first strict minimum (A13)
                nm1[v] = fminf(nm1[v], fmaxf(nm0[v], ax));
                nm0[v] = fminf(nm0[v], ax);
                nloc[v] = lt ? p : nloc[v];
                nib |= (unsigned)(x < 0.f) << v;  // sign(0) = +1
                if (EARLY) syn ^= (unsigned)(sj > 0.f) << v;  // b_j = slice(s_j)
            }
            npar ^= nib;
            unsigned word = nib << sh;
            word |= __shfl_xor_sync(FULL, word, 1);
            word |= __shfl_xor_sync(FULL, word, 2);
            word |= __shfl_xor_sync(FULL, word, 4);
            if ((lane & 7) == 0) SG[(tE + a + p) * 4 + wsel] = word;
        }
        const size_t st = (tm + i) * TILE + 4 * lane;
        const unsigned pc = npar ^ (corr ? 0xfu : 0u);
        float4 o0;
        o0.x = __uint_as_float(__float_as_uint(nm0[0]) | ((pc & 1u) << 31));
        o0.y = __uint_as_float(__float_as_uint(nm0[1]) | (((pc >> 1) & 1u) << 31));
        o0.z = __uint_as_float(__float_as_uint(nm0[2]) | (((pc >> 2) & 1u) << 31));
        o0.w = __uint_as_float(__float_as_uint(nm0[3]) | (((pc >> 3) & 1u) << 31));
        st4(M0 + st, o0);
        st4(M1 + st, make_float4(nm1[0], nm1[1], nm1[2], nm1[3]));
        L4 nl;
        nl.x = (LocT)nloc[0];
        nl.y = (LocT)nloc[1];
        nl.z = (LocT)nloc[2];
        nl.w = (LocT)nloc[3];
        *reinterpret_cast<L4 *>(LC + st) = nl;
        if (EARLY) {
            u0 |= __ballot_sync(FULL, syn & 1u);
            u1 |= __ballot_sync(FULL, syn & 2u);
            u2 |= __ballot_sync(FULL, syn & 4u);
            u3 |= __ballot_sync(FULL, syn & 8u);
        }
        // the generic-proxy reads of buffer b are done before the async proxy refills it
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (q + 2 < nq) stage(q + 2, b);
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
// a5/a6: bit-node sweep of loop body k; stops frames whose b^(k-1) satisfied every check.
// Column edges in chunks of BN_U with all loads of a chunk in flight before the (ordered) sum.
// ------------------------------------------------------------------------------------------------
template <typename LocT, bool EARLY, int BN_U>
__global__ void __launch_bounds__(CTA, BN_U <= 1 ? 6 : MinBlocks<BN_U>::value)
    k_bn(Graph g, StreamState w, int k, int cols_per_cta, int literal, const int *kdev, int check_every) {
    using L4 = typename Vec4<LocT>::type;
    if (kdev) k = *kdev;
    (void)literal;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int T = w.T;
    const int cnt = w.tcount[k & 1];
    if ((int)blockIdx.y >= cnt) return;
    {
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
    const int *__restrict__ col_ptr = g.col_ptr;
    const int4 *__restrict__ bn_edge = g.bn_edge;
    const float *__restrict__ M0 = w.min0;
    const float *__restrict__ M1 = w.min1;
    const LocT *__restrict__ LC = reinterpret_cast<const LocT *>(w.loc);
    const uint32_t *__restrict__ SG = w.sgn;
    const float *__restrict__ R = w.r;
    float *__restrict__ Sv = w.s;
    const int m = g.m, n = g.n, E = g.E;
    const size_t tm = (size_t)t * m, tn = (size_t)t * n, tE = (size_t)t * E;
    const int sh = 4 * (lane & 7), wsel = lane >> 3;
    const int j0 = cblk * cols_per_cta, j1 = min(n, j0 + cols_per_cta);
    for (int j = j0 + warp; j < j1; j += CTA / 32) {
        const int c0 = __ldg(col_ptr + j), dv = __ldg(col_ptr + j + 1) - c0;
        const size_t sj = (tn + j) * TILE + 4 * lane;
        const float4 rv = ld4(R + sj);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        if (BN_U <= 1) {
            for (int q = 0; q < dv; q++) {
                const int4 ed = __ldg(bn_edge + c0 + q);  // {e, i, p, -}, ascending i
                const size_t st = (tm + ed.y) * TILE + 4 * lane;
                const float4 m0 = ld4(M0 + st);
                const float4 m1 = ld4(M1 + st);
                const L4 lc = *reinterpret_cast<const L4 *>(LC + st);
                const unsigned sw = SG[(tE + ed.x) * 4 + wsel] >> sh;
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    const float m0v = comp(m0, v);
                    const float mag = (ed.z == compl4(lc, v)) ? comp(m1, v) : fabsf(m0v);  // Obs. 1
                    const unsigned neg = ((sw >> v) & 1u) ^ (__float_as_uint(m0v) >> 31);   // Obs. 2
                    acc[v] = acc[v] + (neg ? -mag : mag);  // ascending rows from +0.0 (A14)
                }
            }
        } else {
            for (int q0 = 0; q0 < dv; q0 += BN_U) {
                int4 ed[BN_U];
                float4 m0[BN_U], m1[BN_U];
                L4 lc[BN_U];
                unsigned sw[BN_U];
#pragma unroll
                for (int u = 0; u < BN_U; u++)
                    if (q0 + u < dv) ed[u] = __ldg(bn_edge + c0 + q0 + u);
#pragma unroll
                for (int u = 0; u < BN_U; u++) {
                    if (q0 + u < dv) {
                        const size_t st = (tm + ed[u].y) * TILE + 4 * lane;
                        m0[u] = ld4(M0 + st);
                        m1[u] = ld4(M1 + st);
                        lc[u] = *reinterpret_cast<const L4 *>(LC + st);
                        sw[u] = SG[(tE + ed[u].x) * 4 + wsel] >> sh;
                    }
                }
#pragma unroll
                for (int u = 0; u < BN_U; u++) {
                    if (q0 + u >= dv) break;
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        const float m0v = comp(m0[u], v);
                        const float mag = (ed[u].z == compl4(lc[u], v)) ? comp(m1[u], v) : fabsf(m0v);
                        const unsigned neg = ((sw[u] >> v) & 1u) ^ (__float_as_uint(m0v) >> 31);
                        acc[v] = acc[v] + (neg ? -mag : mag);
                    }
                }
            }
        }
        float4 out = make_float4(acc[0] + rv.x, acc[1] + rv.y, acc[2] + rv.z, acc[3] + rv.w);
        if (mine == 0xFu) {
            st4(Sv + sj, out);
        } else if (mine) {
            const float4 old = ld4(Sv + sj);
            out.x = (mine & 1u) ? out.x : old.x;
            out.y = (mine & 2u) ? out.y : old.y;
            out.z = (mine & 4u) ? out.z : old.z;
            out.w = (mine & 8u) ? out.w : old.w;
            st4(Sv + sj, out);
        }
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
__global__ void __launch_bounds__(CTA) k_finalize(StreamState w, int n, int64_t frames, float *__restrict__ post,
                                                  uint8_t *__restrict__ bits) {
    __shared__ float ts[32][TILE + 1];
    __shared__ float tr[32][TILE + 1];
    const int t = blockIdx.y, j0 = blockIdx.x * 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
    for (int fl = warp; fl < TILE; fl += CTA / 32) {
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
        if (lane == 0) {
            if (be) atomicAdd(w.fbe + (size_t)t * TILE + fl, be);
            if (raw) atomicAdd(w.fraw + (size_t)t * TILE + fl, raw);
            if (nz) w.fnz[(size_t)t * TILE + fl] = 1;
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
    if (!run) w.tcount[(L + 1) & 1] = 0;
    cudaGraphSetConditional(h, run ? 1u : 0u);
}

__global__ void k_loop_step(StreamState w, int L, cudaGraphConditionalHandle h) {
    const int k = *w.kdev + 1;
    const bool run = k <= L && w.tcount[k & 1] > 0;
    *w.kdev = k;
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
    if (u >= 4) k_cn<LT, F, EA, 4><<<grid, CTA, 0, st>>>(g, w, k, rpc, lit, kdev);
    else if (u == 2) k_cn<LT, F, EA, 2><<<grid, CTA, 0, st>>>(g, w, k, rpc, lit, kdev);
    else k_cn<LT, F, EA, 1><<<grid, CTA, 0, st>>>(g, w, k, rpc, lit, kdev);
}

template <typename LT, bool EA>
void bn_launch(dim3 grid, cudaStream_t st, const Graph &g, const StreamState &w, int k, int cpc, int lit, int u,
               const int *kdev, int te) {
    if (u >= 2) k_bn<LT, EA, 2><<<grid, CTA, 0, st>>>(g, w, k, cpc, lit, kdev, te);
    else k_bn<LT, EA, 1><<<grid, CTA, 0, st>>>(g, w, k, cpc, lit, kdev, te);
}

template <typename LT, bool F, bool EA>
void cn_tma_launch(const Graph &g, const StreamState &w, int k, int dm, int lit, const int *kdev, cudaStream_t st) {
    const int rpc = (CTA / 32) * ROWS_PER_WARP;
    const dim3 grid = grid2((g.m + rpc - 1) / rpc, w.T);
    const size_t smem = (size_t)(CTA / 32) * 2 * cn_stage_bytes(dm, (int)sizeof(LT));
    cudaFuncSetAttribute(k_cn_tma<LT, F, EA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_cn_tma<LT, F, EA><<<grid, CTA, smem, st>>>(g, w, k, dm, lit, kdev);
}

int launch_check_node(const Graph &g, const StreamState &w, int k, bool first, bool early, bool literal, bool loc16,
                      const StreamLaunch &cfg, cudaStream_t st, const int *kdev) {
    if (cfg.cn_tma_dm > 0) {  // bulk-copy staged variant
        const int dm = cfg.cn_tma_dm, lit = literal ? 1 : 0;
        if (loc16) {
            if (first) { if (early) cn_tma_launch<uint16_t, true, true>(g, w, k, dm, lit, kdev, st);
                         else cn_tma_launch<uint16_t, true, false>(g, w, k, dm, lit, kdev, st); }
            else { if (early) cn_tma_launch<uint16_t, false, true>(g, w, k, dm, lit, kdev, st);
                   else cn_tma_launch<uint16_t, false, false>(g, w, k, dm, lit, kdev, st); }
        } else {
            if (first) { if (early) cn_tma_launch<uint8_t, true, true>(g, w, k, dm, lit, kdev, st);
                         else cn_tma_launch<uint8_t, true, false>(g, w, k, dm, lit, kdev, st); }
            else { if (early) cn_tma_launch<uint8_t, false, true>(g, w, k, dm, lit, kdev, st);
                   else cn_tma_launch<uint8_t, false, false>(g, w, k, dm, lit, kdev, st); }
        }
        return 1;
    }
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
    const dim3 grid = grid2((g.n + cfg.cols_per_cta - 1) / cfg.cols_per_cta, w.T);
    const int lit = literal ? 1 : 0, cpc = cfg.cols_per_cta, u = cfg.bn_unroll;
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
    k_finalize<<<grid2((g.n + 31) / 32, w.T), CTA, 0, st>>>(w, g.n, frames, posterior, bits);
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
