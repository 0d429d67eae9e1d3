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
// warp owns frames ("slots") 4l..4l+3, so every gather of s, r or row state is one 512-byte
// contiguous float4 access per warp, and per-slot bits of 128 slots are four ballot words.
//
// Row record of row i in tile t (rs bytes, 32-byte aligned; see ldpc_internal.cuh):
//   [0, 512)            min0 [128] fp32  |lambda| minimum; SIGN BIT = row sign parity x (-1)^{d_i} (A1)
//   [512, 1024)         min1 [128] fp32  second minimum (Obs. 1), same sign bit
//   [1024 + 32 p, +32)  edge p of N_i: byte l = sign nibble (bit v = sign of lambda_e for slot 4l+v)
//                                      | isloc nibble << 4 (bit v: p == min0Location of slot 4l+v)
// eta_e = (isloc ? min1 : min0) with its sign bit XORed with the stored sign: one SEL and one LOP3 per
// frame-edge.  The bit node gathers per edge 512 + 512 + 32 bytes per warp (the edge's own 32-byte
// block, not a whole row of locations and sign words).
//
// Sweeps are persistent grids that take (tile, block) items from a work counter, so a sweep over a
// handful of still-running tiles costs no empty CTAs.  Early stop is exact per frame; the work is
// per tile, and tiles whose running frames fall under half are COMPACTED: their
// running frames are moved, with their whole state, into fresh dense tiles at the end of the
// workspace, so a tile stops costing its slowest frame.  Every slot carries its frame index, and the
// outputs are written through it at the end.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "ldpc_internal.cuh"

#include <type_traits>

namespace ldpc {

namespace {

constexpr unsigned FULL_MASK = 0xffffffffu;

__device__ __forceinline__ float comp(const float4 &a, int v) { return v == 0 ? a.x : v == 1 ? a.y : v == 2 ? a.z : a.w; }
__device__ __forceinline__ unsigned comp(const uint4 &a, int v) { return v == 0 ? a.x : v == 1 ? a.y : v == 2 ? a.z : a.w; }
__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ void st4(float *p, float4 v) { *reinterpret_cast<float4 *>(p) = v; }
__device__ __forceinline__ uint4 ldu4(const uint32_t *p) { return *reinterpret_cast<const uint4 *>(p); }

// L2 eviction priorities (createpolicy + .L2::cache_hint; the policy sits in the load's uniform descriptor,
// no per-access cost).  Bit 0: data read or written once per sweep (r, s stores, the check node's row
// records) is marked evict_first; bit 1: data gathered several times per sweep (s in the check node, row
// records in the bit node) evict_last, so a tile's gathered working set stays in L2 while it is swept.
// Measured (8192 frames, every frame running): bit node bits 0+1: C4 -2.5 % (DRAM / algorithmic bytes
// 1.18 -> 1.02), C3 equal; check node bit 1 (s gathers evict_last): C3 -2.2 %, C4 -1.5 %, while bit 0 on
// its row records costs 1-1.5 %.
#ifndef L2H_CN
#define L2H_CN 2
#endif
#ifndef L2H_BN
#define L2H_BN 3
#endif
__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
template <int BIT, int L2H>
__device__ __forceinline__ float4 ldh4(const float *p, uint64_t pol) {
    if (!(L2H & BIT)) return *reinterpret_cast<const float4 *>(p);
    float4 v;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
template <int BIT, int L2H>
__device__ __forceinline__ void sth4(float *p, float4 v, uint64_t pol) {
    if (!(L2H & BIT)) {
        *reinterpret_cast<float4 *>(p) = v;
        return;
    }
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w), "l"(pol)
                 : "memory");
}

// min(a, b, c) in one FMNMX3 (sm_100)
__device__ __forceinline__ float fmin3f(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// check node: edges in pairs (FMNMX3 second-minimum update, 3-input parity XOR).  k_cn (rows of degree
// <= 8): no gain (C3 -0.5 %, C4 equal) and 1-2 % more SASS (selects of the half-empty last pair), so off;
// k_cn_generic (C6, d = 32): -4 %, on.
#ifndef CN_PAIR
#define CN_PAIR 0
#endif
#ifndef CNG_PAIR
#define CNG_PAIR 1
#endif
// check node (k_cn): min0 / min1 by a pair tournament after all of a row's lambdas, min0Location as the
// edges that attain min0 (see cn_compute); 0: first-strict-minimum tracking edge by edge
#ifndef CN_TREE
#define CN_TREE 1
#endif
#ifndef CNG_TREE
#define CNG_TREE 1  // the same for each 8-edge chunk of k_cn_generic (rows of at most 8 NWK edges)
#endif

// 256-bit (8 x fp32) global accesses (LDG.E.ENL2.256 / STG.E.ENL2.256 on sm_100), with an optional L2 policy
struct f8 {
    float v[8];
};
template <int L2H>
__device__ __forceinline__ f8 ld8h(const float *p, uint64_t pol) {
    f8 r;
    if (L2H)
        asm volatile("ld.global.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                       "=f"(r.v[6]), "=f"(r.v[7])
                     : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                       "=f"(r.v[6]), "=f"(r.v[7])
                     : "l"(p));
    return r;
}
template <int L2H>
__device__ __forceinline__ void st8h(float *p, const f8 &r, uint64_t pol) {
    if (L2H)
        asm volatile("st.global.L2::cache_hint.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(p), "f"(r.v[0]),
                     "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7]), "l"(pol)
                     : "memory");
    else
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]),
                     "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7])
                     : "memory");
}

// the sign of a magnitude picked by Obs. 1 flipped by one stored sign bit (already moved to bit 31)
__device__ __forceinline__ float flip31(float mag, uint32_t bit31) {
    return __uint_as_float(__float_as_uint(mag) ^ (bit31 & 0x80000000u));
}

// CTA barrier reached by every thread, with the warp reconverged first (barrier.sync is .aligned: the
// whole warp must execute it together; the per-lane branches before it need not reconverge on their own)
__device__ __forceinline__ void cta_sync() {
    __syncwarp();
    __syncthreads();
}

// zeros of s and r are kept as -0 in the streaming schedule (reading A12: same slice and sign())
__device__ __forceinline__ float zneg(float x) { return x == 0.f ? -0.0f : x; }

// Take the next (tile, block) item of a persistent sweep from a work counter.  Two barriers: every
// thread has finished the previous item (and read its index) before thread 0 overwrites s_item.
__device__ __forceinline__ int next_item(int *ctr, int &s_item) {
    cta_sync();
    if (threadIdx.x == 0) s_item = atomicAdd(ctr, 1);
    cta_sync();
    return s_item;
}

#ifndef CN_T
#define CN_T 256
#endif
#ifndef CN_MINB
#define CN_MINB 3
#endif
#ifndef CN_PF
#define CN_PF 0  // 1: prefetch the next row's gathers and state into L1 while the current row is computed
#endif
#ifndef CNG_MINB
#define CNG_MINB 2  // any-degree check node: CTAs of CN_T threads per SM (2: 128 registers)
#endif
#ifndef CNG_PF
#define CNG_PF 1  // any-degree check node: the next chunk's gathers prefetched into L1 (C6: -8 %)
#endif
#ifndef CN_SMEMU
#define CN_SMEMU 0  // 1: syndrome ballots OR-ed into shared memory per row instead of per-item registers
#endif
#ifndef BN_T
#define BN_T 128  // the bit node lives on loads in flight
#endif
#ifndef BN_MINB
#define BN_MINB 12  // 12 x 128 threads (48 warps per SM)
#endif
#ifndef CN_ROWS_N
#define CN_ROWS_N 128
#endif
constexpr int CN_ROWS = CN_ROWS_N;  // rows per check-node item (16 per warp; at most 32 per warp)
// rows per item of the any-degree check node: 64 (8 per warp) -- C6 (1022 rows of degree 32) check node
// -14.7 % against 128 (8192 frames, every frame running: twice the items, shorter tail); 64 and 256 rows
// per item in k_cn measured equal or 1-7 % slower (C3, C4)
#ifndef CNG_ROWS_N
#define CNG_ROWS_N 64
#endif
constexpr int CNG_ROWS = CNG_ROWS_N;
#ifndef BN_COLS
#define BN_COLS 16  // columns per bit-node item (4 per warp)
#endif
constexpr int CN_NW = CN_T / 32;

// ------------------------------------------------------------------------------------------------
// a2: stage-in.  llr [F][n] -> r [t][n][128] (zeros kept as -0: same slice and sign() under reading
// A12; with every zero of r and s being -0, slice(s) = 0 iff the IEEE sign bit of s is set), the
// per-slot frame index, per-tile flags, and the raw channel errors of every frame (r_j > 0) counted
// where r is read anyway.  Body 1 reads r itself (s = r).
// ------------------------------------------------------------------------------------------------
constexpr int SI_SUB = 8;  // 32-column sub-blocks per stage-in / finalize CTA

__global__ void __launch_bounds__(CTA) k_stage_in(const float *__restrict__ llr, int64_t frames, int n,
                                                  StreamState w) {
    __shared__ float tile[32][TILE + 1];
    const int t = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t f0 = (int64_t)t * TILE;
    int raw = 0;  // lane q < 16 of warp w counts frame w + 8q
    for (int sb = 0; sb < SI_SUB; sb++) {
        const int j0 = (blockIdx.x * SI_SUB + sb) * 32;
        if (j0 >= n) break;
        const int j = j0 + lane;
        for (int fl = warp; fl < TILE; fl += CTA / 32) {
            const int64_t f = f0 + fl;
            const bool ok = f < frames && j < n;
            const float v = ok ? __ldg(llr + f * n + j) : -1.0f;
            tile[lane][fl] = v;
            const int c = __popc(__ballot_sync(FULL_MASK, ok && v > 0.f));
            if (lane == (fl >> 3)) raw += c;
        }
        cta_sync();
        for (int jl = warp; jl < 32; jl += CTA / 32) {
            const int jj = j0 + jl;
            if (jj >= n) break;
            const size_t base = ((size_t)t * n + jj) * TILE;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const float v = tile[jl][lane + 32 * q];
                w.r[base + lane + 32 * q] = v == 0.f ? -0.0f : v;  // zeros kept as -0 (reading A12)
            }
        }
        cta_sync();
    }
    if (lane < 16 && raw) {
        const int64_t f = f0 + warp + 8 * lane;
        if (f < frames) atomicAdd(w.fraw + f, raw);
    }
    if (blockIdx.x == 0) {
        const int tid = threadIdx.x;
        if (tid < 4) {
            // slot 4*lane+v of the tile is bit `lane` of word v; padding slots start "done"
            uint32_t pad = 0;
            for (int l = 0; l < 32; l++)
                if (f0 + 4 * l + tid >= frames) pad |= 1u << l;
            w.done[(size_t)t * 4 + tid] = pad;
            w.unsat[(size_t)t * 4 + tid] = 0;
            w.unsat[((size_t)w.Tcap + t) * 4 + tid] = 0;
        }
        if (tid < TILE) w.fid[(size_t)t * TILE + tid] = (f0 + tid < frames) ? (int)(f0 + tid) : -1;
        if (tid == 0) {
            w.tlist[(size_t)w.Tcap + t] = t;  // body 1 runs every tile
            if (t == 0) {
                w.tcount[0] = 0;
                w.tcount[1] = w.T;
                w.work[WK_CN] = 0;
                w.work[WK_BN] = 0;
                w.work[WK_MOVE] = 0;
                w.work[WK_SYN] = 0;
                w.ctl[CT_TNEXT] = w.T;
                w.ctl[CT_NSRC] = 0;
                w.ctl[CT_NDST] = 0;
            }
        }
    }
}

// ------------------------------------------------------------------------------------------------
// a3/a4/a6: check-node sweep of loop body k (k = 1..L), fused syndrome of b^(k-1).
// FIRST: eta^prev = 0, no old state is read, lambda = r.
// A warp owns rows i0 + warp + 8q of its item.  Per row, every load -- the CH gathers of s (512-byte
// float4 segments, lane = 4 slots), the row's min0/min1 and the lane's old edge bytes -- is issued
// before any arithmetic, and the column indices of the next row are fetched meanwhile, so each row
// costs one memory latency, overlapped across the warps of the SM.  All loads are unconditional
// (edges past d_i read column 0 of the tile; the record holds CH edge blocks).
// Per frame-edge: eta^prev = (isloc ? min1 : min0) ^ sign (SHF, ISETP, SEL, LOP3), lambda (FADD),
// first-strict-minimum tracking (FSETP, 3 FMNMX, SEL; reading A13), the new sign bit, and, when
// EARLY, the decision parity (slice(s) = 0 iff bit 31 of bits(s) - 1 is set, s never -0).
// ------------------------------------------------------------------------------------------------
template <int CH>
struct CnRow {
    float4 sv[CH];
    float4 m0, m1;
    uint32_t eb[CH];
};

__device__ __forceinline__ void pf_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// L1 prefetch of a row's loads (no registers held across the latency): its CH gathers and its state
template <int CH, bool FIRST>
__device__ __forceinline__ void cn_prefetch(int cj, const float *__restrict__ Sl, const unsigned char *__restrict__ Ri,
                                            int lane) {
    if (!FIRST) {
        pf_l1(reinterpret_cast<const float *>(Ri) + 4 * lane);
        pf_l1(reinterpret_cast<const float *>(Ri) + 128 + 4 * lane);
    }
#pragma unroll
    for (int u = 0; u < CH; u++) pf_l1(Sl + (size_t)__shfl_sync(FULL_MASK, cj, u) * TILE);
}

template <int CH, bool FIRST>
__device__ __forceinline__ void cn_fetch(CnRow<CH> &R, int cj, const float *__restrict__ Sl,
                                         const unsigned char *__restrict__ Ri, int lane, uint64_t pf, uint64_t pl) {
    if (!FIRST) {
        R.m0 = ldh4<1, L2H_CN>(reinterpret_cast<const float *>(Ri) + 4 * lane, pf);
        R.m1 = ldh4<1, L2H_CN>(reinterpret_cast<const float *>(Ri) + 128 + 4 * lane, pf);
#pragma unroll
        for (int p = 0; p < CH; p++) R.eb[p] = Ri[REC_EDGE0 + 32 * p + lane];
    }
#pragma unroll
    for (int u = 0; u < CH; u++) {
        const int j = __shfl_sync(FULL_MASK, cj, u);
        R.sv[u] = ldh4<2, L2H_CN>(Sl + (size_t)j * TILE, pl);
    }
}

// FULL: the row has exactly CH edges (no per-edge guard).  Per frame-edge on the ALU pipe: the isloc
// test and magnitude select (2), the sign flip (1), the decision parity (1, zeros of s are -0: slice(s)
// = 0 iff the IEEE sign bit is set), first-strict-minimum tracking (FSETP, 3 FMNMX, SEL; reading A13)
// and the new sign bit (one funnel shift).  lambda = (s - eta) + 0 runs on the otherwise idle FMA pipe
// and makes every zero lambda +0, so its sign (sign(0) = +1) is its IEEE sign bit.
template <int CH, bool FIRST, bool EARLY, bool FULL>
__device__ __forceinline__ void cn_compute(const CnRow<CH> &R, unsigned char *__restrict__ Ri, int d, int literal,
                                           int lane, uint32_t (&u)[4], uint32_t *su, uint64_t pf) {
    const float INF = __int_as_float(0x7f800000);
    const float om0[4] = {R.m0.x, R.m0.y, R.m0.z, R.m0.w}, om1[4] = {R.m1.x, R.m1.y, R.m1.z, R.m1.w};
    float nm0[4] = {INF, INF, INF, INF}, nm1[4] = {INF, INF, INF, INF};
#if !CN_TREE || CN_PAIR
    int nloc[4] = {0, 0, 0, 0};
#endif
    uint32_t syn[4] = {0u, 0u, 0u, 0u}, sw = 0;  // sw: sign bits pushed in (p, v) order
#if CN_PAIR
    // Edges in pairs (p, p+1): the pair's smaller and larger |lambda| (s, t) update the row state with
    //   nm0' = min(nm0, s), nm1' = min3(nm1, max(nm0, s), t) (FMNMX3), loc' = s < nm0 ? (t-edge < s-edge ?
    //   p+1 : p) : loc -- the same first strict minimum (A13) and second minimum as the edge-by-edge update,
    // in 9 instead of 10 ALU operations per pair and slot; the decision parity takes both edges in one
    // 3-input XOR.  An edge past d_i enters as |lambda| = +inf and parity 0 (it changes nothing).
#pragma unroll
    for (int p = 0; p < CH; p += 2) {
        const bool va = FULL || p < d, vb = p + 1 < CH && (FULL || p + 1 < d);
        if (!va) continue;
        const uint32_t ba = FIRST ? 0u : R.eb[p], bb = (FIRST || p + 1 >= CH) ? 0u : R.eb[p + 1];
        float xa[4], xb[4];
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const float sa = comp(R.sv[p], v);
            const float sb = p + 1 < CH ? comp(R.sv[p + 1], v) : 0.f;
            if (FIRST) {
                xa[v] = __fadd_rn(sa, 0.0f);  // eta^prev = 0
                xb[v] = __fadd_rn(sb, 0.0f);
            } else {
                const float ma = (ba & (16u << v)) ? om1[v] : om0[v];  // Obs. 1 (+ row parity)
                const float mb = (bb & (16u << v)) ? om1[v] : om0[v];
                xa[v] = __fadd_rn(__fsub_rn(sa, flip31(ma, ba << (31 - v))), 0.0f);  // lambda - eta^prev
                xb[v] = __fadd_rn(__fsub_rn(sb, flip31(mb, bb << (31 - v))), 0.0f);
            }
            if (EARLY) syn[v] ^= __float_as_uint(sa) ^ (vb ? __float_as_uint(sb) : 0u);  // bit 31: slice(s_j) == 0
        }
#pragma unroll
        for (int v = 0; v < 4; v++) sw = __funnelshift_l(__float_as_uint(xa[v]), sw, 1);
        if (vb) {
#pragma unroll
            for (int v = 0; v < 4; v++) sw = __funnelshift_l(__float_as_uint(xb[v]), sw, 1);
        }
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const float a = fabsf(xa[v]), b = vb ? fabsf(xb[v]) : INF;
            const float sm = fminf(a, b), tm = fmaxf(a, b);
            const int lp = b < a ? p + 1 : p;
            const bool lt = sm < nm0[v];
            nm1[v] = fmin3f(nm1[v], fmaxf(nm0[v], sm), tm);
            nm0[v] = fminf(nm0[v], sm);
            nloc[v] = lt ? lp : nloc[v];
        }
    }
#elif CN_TREE
    // Every lambda of the row first, then min0 / min1 by a pair tournament and min0Location as the edges
    // whose |lambda| equals min0.  The tournament keeps (lo, hi) = the two smallest |lambda| seen: a pair
    // (a, b) enters as (min, max) and merges by lo' = min(lo, l2), hi' = min3(hi, h2, max(lo, l2)) -- 2.1
    // FMNMX per slot-edge for CH = 7 instead of FSETP + 3 FMNMX + SEL.  isloc_p = (|lambda_p| == min0)
    // marks every edge of a tie; under a tie min1 = min0 (same value, same sign bit), so eta_e =
    // (isloc ? min1 : min0) is the same value as with the first strict minimum only (reading A13).  Its
    // bit is the complement of the sign bit of min0 - |lambda_p| (exact, +0 iff equal; an FMA-pipe
    // FADD), pushed like the sign bits.  Edges past d_i enter as |lambda| = +inf (never a minimum, never
    // a location); their pushed sign bits are masked off.
    float ax[CH][4];
    uint32_t iw = 0;
#pragma unroll
    for (int p = 0; p < CH; p++) {
        const bool va = FULL || p < d;
        const uint32_t b = FIRST ? 0u : R.eb[p];
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const float sj = comp(R.sv[p], v);
            float x;
            if (FIRST) {
                x = __fadd_rn(sj, 0.0f);  // eta^prev = 0
            } else {
                const float mag = (b & (16u << v)) ? om1[v] : om0[v];  // Obs. 1 (+ row parity)
                x = __fadd_rn(__fsub_rn(sj, flip31(mag, b << (31 - v))), 0.0f);  // lambda - eta^prev
            }
            ax[p][v] = va ? fabsf(x) : INF;
            sw = __funnelshift_l(__float_as_uint(x), sw, 1);
            if (EARLY) syn[v] ^= va ? __float_as_uint(sj) : 0u;  // bit 31: slice(s_j) == 0
        }
    }
#pragma unroll
    for (int v = 0; v < 4; v++) {
        float lo = fminf(ax[0][v], ax[1][v]), hi = fmaxf(ax[0][v], ax[1][v]);
#pragma unroll
        for (int p = 2; p + 1 < CH; p += 2) {
            const float l2 = fminf(ax[p][v], ax[p + 1][v]), h2 = fmaxf(ax[p][v], ax[p + 1][v]);
            hi = fmin3f(hi, h2, fmaxf(lo, l2));
            lo = fminf(lo, l2);
        }
        if (CH & 1) {
            hi = fminf(hi, fmaxf(lo, ax[CH - 1][v]));
            lo = fminf(lo, ax[CH - 1][v]);
        }
        nm0[v] = lo;
        nm1[v] = hi;
    }
#pragma unroll
    for (int p = 0; p < CH; p++)
#pragma unroll
        for (int v = 0; v < 4; v++) iw = __funnelshift_l(__float_as_uint(__fsub_rn(nm0[v], ax[p][v])), iw, 1);
#else
#pragma unroll
    for (int p = 0; p < CH; p++) {
        if (FULL || p < d) {
            const uint32_t b = FIRST ? 0u : R.eb[p];
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const float sj = comp(R.sv[p], v);
                float x;
                if (FIRST) {
                    x = __fadd_rn(sj, 0.0f);  // eta^prev = 0
                } else {
                    const float mag = (b & (16u << v)) ? om1[v] : om0[v];  // Obs. 1 (+ row parity)
                    x = __fadd_rn(__fsub_rn(sj, flip31(mag, b << (31 - v))), 0.0f);  // lambda - eta^prev
                }
                const float ax = fabsf(x);
                const bool lt = ax < nm0[v];  // first strict minimum (A13)
                nm1[v] = fminf(nm1[v], fmaxf(nm0[v], ax));
                nm0[v] = fminf(nm0[v], ax);
                nloc[v] = lt ? p : nloc[v];
                if (EARLY) syn[v] ^= __float_as_uint(sj);  // bit 31: slice(s_j) == 0
                sw = __funnelshift_l(__float_as_uint(x), sw, 1);
            }
        }
    }
#endif
    // bit 4p+v of sw = sign of lambda (edge p, slot 4l+v)
#if CN_TREE && !CN_PAIR
    sw = CH == 8 ? __brev(sw) : __brev(sw) >> (32 - 4 * CH);
    if (!FULL) sw &= (1u << (4 * d)) - 1u;  // d < CH <= 8
    const uint32_t lm = CH == 8 ? __brev(~iw) : __brev(~iw) >> (32 - 4 * CH);  // bit 4p+v: isloc
#else
    if (FULL) sw = CH == 8 ? __brev(sw) : __brev(sw) >> (32 - 4 * CH);
    else sw = __brev(sw) >> (32 - 4 * d);
#endif
    // sign parity per slot (Obs. 2): XOR of bits v, v+4, ..., of sw, times (-1)^{d_i} (reading A1)
    uint32_t pw = sw ^ (sw >> 16);
    pw ^= pw >> 8;
    pw ^= pw >> 4;
    pw ^= ((uint32_t)(d & 1) & (uint32_t)(!literal)) ? 0xfu : 0u;
    const uint32_t s0 = pw << 31, s1 = (pw << 30) & 0x80000000u, s2 = (pw << 29) & 0x80000000u,
                   s3 = (pw << 28) & 0x80000000u;
    sth4<1, L2H_CN>(reinterpret_cast<float *>(Ri) + 4 * lane,
            make_float4(__uint_as_float(__float_as_uint(nm0[0]) | s0), __uint_as_float(__float_as_uint(nm0[1]) | s1),
                        __uint_as_float(__float_as_uint(nm0[2]) | s2), __uint_as_float(__float_as_uint(nm0[3]) | s3)),
            pf);
    sth4<1, L2H_CN>(reinterpret_cast<float *>(Ri) + 128 + 4 * lane,
            make_float4(__uint_as_float(__float_as_uint(nm1[0]) | s0), __uint_as_float(__float_as_uint(nm1[1]) | s1),
                        __uint_as_float(__float_as_uint(nm1[2]) | s2), __uint_as_float(__float_as_uint(nm1[3]) | s3)),
            pf);
    // edge bytes: sign nibble | isloc nibble << 4.  lm has bit 4p+v set iff min0Location of slot v is p;
    // interleaving the nibbles of sw and lm gives the bytes of the even edges in ze, of the odd ones in zo
#if !CN_TREE || CN_PAIR
    const uint32_t lm = (1u << (4 * nloc[0])) | (2u << (4 * nloc[1])) | (4u << (4 * nloc[2])) | (8u << (4 * nloc[3]));
#endif
    const uint32_t ze = (sw & 0x0f0f0f0fu) | ((lm & 0x0f0f0f0fu) << 4);
    const uint32_t zo = ((sw >> 4) & 0x0f0f0f0fu) | (lm & 0xf0f0f0f0u);
#pragma unroll
    for (int p = 0; p < CH; p++)
        if (FULL || p < d) Ri[REC_EDGE0 + 32 * p + lane] = (unsigned char)(((p & 1) ? zo : ze) >> (8 * (p >> 1)));
    if (EARLY) {
        const uint32_t dp = (uint32_t)(d & 1);  // XOR_j b_j = d_i mod 2 xor XOR_j (1 - b_j)
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const uint32_t bv = __ballot_sync(FULL_MASK, ((syn[v] >> 31) ^ dp) != 0u);
            if (CN_SMEMU) {  // straight into the CTA's words (4 registers fewer across the row loop)
                if (lane == 0 && bv) atomicOr(su + v, bv);
            } else {
                u[v] |= bv;
            }
        }
    }
}

// Rows of degree up to 8 (CH = the smallest instance >= the maximum row degree).
template <int CH, bool FIRST, bool EARLY>
__global__ void __launch_bounds__(CN_T, CN_MINB) k_cn(Graph g, StreamState w, int k, int literal, const int *kdev) {
    if (kdev) k = *kdev;  // body index supplied by the graph-driven loop
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t s_u[4];
    __shared__ int s_item;
    const int cnt = w.tcount[k & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        w.tcount[(k + 1) & 1] = 0;  // rebuilt by k_bn of body k
        w.work[WK_BN] = 0;
        w.ctl[CT_NSRC] = 0;
        if (w.nlaunch) w.nlaunch[4] += (unsigned long long)cnt;  // tile-bodies swept by the check node
    }
    const int m = g.m, n = g.n;
    const int nrb = (m + CN_ROWS - 1) / CN_ROWS;
    const int items = cnt * nrb;
    const uint64_t pf = (L2H_CN & 1) ? pol_first() : 0, pl = (L2H_CN & 2) ? pol_last() : 0;
    for (;;) {
        if (EARLY && threadIdx.x < 4) s_u[threadIdx.x] = 0;
        const int it = next_item(w.work + WK_CN, s_item);
        if (it >= items) break;
        const int y = it / nrb, x = it - y * nrb;
        const int t = w.tlist[(size_t)(k & 1) * w.Tcap + y];
        const float *__restrict__ Sl = (FIRST ? w.r : w.s) + (size_t)t * n * TILE + 4 * lane;
        unsigned char *RB = w.rst + (size_t)t * m * w.rs;
        const int i0 = x * CN_ROWS + warp, i1 = min(m, x * CN_ROWS + CN_ROWS);
        const int nr = i0 < i1 ? (i1 - i0 + CN_NW - 1) / CN_NW : 0;  // rows of this warp (<= 16)
        uint32_t u[4] = {0u, 0u, 0u, 0u};
        if (nr > 0) {
            int ra = 0, rb = 0;  // lane q: row_ptr of the warp's row q
            if (lane < nr) {
                ra = __ldg(g.row_ptr + i0 + CN_NW * lane);
                rb = __ldg(g.row_ptr + i0 + CN_NW * lane + 1);
            }
            auto cols_of = [&](int q) {  // lane p: column of edge p of row q (0 past the degree / the rows)
                const int a = __shfl_sync(FULL_MASK, ra, q & 31), d = __shfl_sync(FULL_MASK, rb, q & 31) - a;
                return (q < nr && lane < d) ? __ldg(g.col_idx + a + lane) : 0;
            };
            CnRow<CH> A;
            int cj = cols_of(0);
            for (int q = 0; q < nr; q++) {
                const int i = i0 + CN_NW * q;
                unsigned char *Ri = RB + (size_t)i * w.rs;
                cn_fetch<CH, FIRST>(A, cj, Sl, Ri, lane, pf, pl);
                const int d = __shfl_sync(FULL_MASK, rb, q) - __shfl_sync(FULL_MASK, ra, q);
                cj = cols_of(q + 1);
                if (CN_PF && q + 1 < nr) cn_prefetch<CH, FIRST>(cj, Sl, RB + (size_t)(i + CN_NW) * w.rs, lane);
                if (d == CH) cn_compute<CH, FIRST, EARLY, true>(A, Ri, d, literal, lane, u, s_u, pf);
                else cn_compute<CH, FIRST, EARLY, false>(A, Ri, d, literal, lane, u, s_u, pf);
            }
        }
        if (EARLY) {
            if (lane == 0) {
#pragma unroll
                for (int v = 0; v < 4; v++)
                    if (u[v]) atomicOr(&s_u[v], u[v]);
            }
            cta_sync();
            if (threadIdx.x < 4 && s_u[threadIdx.x])
                atomicOr(w.unsat + ((size_t)(k & 1) * w.Tcap + t) * 4 + threadIdx.x, s_u[threadIdx.x]);
        }
    }
}

// Rows of any degree: edges in chunks of 8 (one gather batch, all loads in flight together).  The sign
// bits of a chunk are pushed into one word by a funnel shift per frame-edge and its edge bytes written at
// the end of the chunk; NWK > 0 (rows of at most 8*NWK edges) keeps the chunk words in registers and
// merges the isloc nibbles into the bytes of the min0Location edges at the end of the row; NWK = 0 (any
// degree) ORs them into the bytes already written (each lane owns byte `lane` of every edge block).
template <bool FIRST, bool EARLY, int NWK>
__global__ void __launch_bounds__(CN_T, CNG_MINB) k_cn_generic(Graph g, StreamState w, int k, int literal, const int *kdev) {
    if (kdev) k = *kdev;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t s_u[4];
    __shared__ int s_item;
    const int cnt = w.tcount[k & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        w.tcount[(k + 1) & 1] = 0;
        w.work[WK_BN] = 0;
        w.ctl[CT_NSRC] = 0;
        if (w.nlaunch) w.nlaunch[4] += (unsigned long long)cnt;
    }
    const int m = g.m, n = g.n;
    const int nrb = (m + CNG_ROWS - 1) / CNG_ROWS;
    const int items = cnt * nrb;
    const float INF = __int_as_float(0x7f800000);
    constexpr int C8 = 8;
    for (;;) {
        if (EARLY && threadIdx.x < 4) s_u[threadIdx.x] = 0;
        const int it = next_item(w.work + WK_CN, s_item);
        if (it >= items) break;
        const int y = it / nrb, x = it - y * nrb;
        const int t = w.tlist[(size_t)(k & 1) * w.Tcap + y];
        const float *__restrict__ Sl = (FIRST ? w.r : w.s) + (size_t)t * n * TILE + 4 * lane;
        unsigned char *RB = w.rst + (size_t)t * m * w.rs;
        uint32_t u[4] = {0u, 0u, 0u, 0u};
        // the warp's rows i0 + 8q: their row pointers in lanes q (one load), and the first 32 column
        // indices of the next row fetched while the current row is processed
        const int i0 = x * CNG_ROWS + warp, i1 = min(m, x * CNG_ROWS + CNG_ROWS);
        const int nr = i0 < i1 ? (i1 - i0 + CN_NW - 1) / CN_NW : 0;
        int ra = 0, rb = 0;
        if (lane < nr) {
            ra = __ldg(g.row_ptr + i0 + CN_NW * lane);
            rb = __ldg(g.row_ptr + i0 + CN_NW * lane + 1);
        }
        int cj_next = 0;
        if (nr > 0) {
            const int a0 = __shfl_sync(FULL_MASK, ra, 0), d0 = __shfl_sync(FULL_MASK, rb, 0) - a0;
            cj_next = lane < d0 ? __ldg(g.col_idx + a0 + lane) : 0;
        }
        for (int q = 0; q < nr; q++) {
            const int i = i0 + CN_NW * q;
            const int a = __shfl_sync(FULL_MASK, ra, q), d = __shfl_sync(FULL_MASK, rb, q) - a;
            const int cj_row = cj_next;
            {
                const int an = __shfl_sync(FULL_MASK, ra, (q + 1) & 31), dn = __shfl_sync(FULL_MASK, rb, (q + 1) & 31) - an;
                cj_next = (q + 1 < nr && lane < dn) ? __ldg(g.col_idx + an + lane) : 0;
            }
            unsigned char *Ri = RB + (size_t)i * w.rs;
            float om0[4] = {0.f, 0.f, 0.f, 0.f}, om1[4] = {0.f, 0.f, 0.f, 0.f};
            if (!FIRST) {
                const float4 A = ld4(reinterpret_cast<const float *>(Ri) + 4 * lane);
                const float4 B = ld4(reinterpret_cast<const float *>(Ri) + 128 + 4 * lane);
                om0[0] = A.x; om0[1] = A.y; om0[2] = A.z; om0[3] = A.w;
                om1[0] = B.x; om1[1] = B.y; om1[2] = B.z; om1[3] = B.w;
            }
            float nm0[4] = {INF, INF, INF, INF}, nm1[4] = {INF, INF, INF, INF};
            int nloc[4] = {0, 0, 0, 0};
            uint32_t syn[4] = {0u, 0u, 0u, 0u}, pf = 0u;
            uint32_t cws[NWK > 0 ? NWK : 1];
#if CNG_TREE
            float clo[NWK > 0 ? NWK : 1][4];  // chunk minima per slot
            uint32_t cls[NWK > 0 ? NWK : 1];  // chunk isloc candidates (bit 4u+v)
#endif
            int cj = cj_row;
            // NWK > 0: the chunk loop is unrolled (chunk words stay in registers)
#pragma unroll(NWK > 0 ? NWK : 1)
            for (int p0 = 0; p0 < (NWK > 0 ? 8 * NWK : d); p0 += C8) {
                if (NWK > 0 && p0 >= d) break;
                if (p0 > 0 && (p0 & 31) == 0) cj = (lane < d - p0) ? __ldg(g.col_idx + a + p0 + lane) : 0;
                const bool full = p0 + C8 <= d;  // warp-uniform
                float4 sv[C8];
                uint32_t eb[C8];
#pragma unroll
                for (int u8 = 0; u8 < C8; u8++) {
                    const int j = __shfl_sync(FULL_MASK, cj, (p0 + u8) & 31);
                    sv[u8] = ld4(Sl + (size_t)j * TILE);  // unconditional: edges past d_i read column 0
                    eb[u8] = FIRST ? 0u : Ri[REC_EDGE0 + 32 * (p0 + u8) + lane];
                }
                if (CNG_PF) {  // the next chunk's gathers into L1 while this chunk is computed
                    if (p0 + C8 < d && ((p0 + C8) & 31) != 0) {
#pragma unroll
                        for (int u8 = 0; u8 < C8; u8++) pf_l1(Sl + (size_t)__shfl_sync(FULL_MASK, cj, (p0 + C8 + u8) & 31) * TILE);
                    } else if (p0 + C8 >= d && q + 1 < nr) {  // last chunk: the next row's first chunk
#pragma unroll
                        for (int u8 = 0; u8 < C8; u8++) pf_l1(Sl + (size_t)__shfl_sync(FULL_MASK, cj_next, u8) * TILE);
                    }
                }
                uint32_t cw = 0;
#if CNG_TREE
                if constexpr (NWK > 0) {
                    // the chunk's lambdas first, then its two smallest |lambda| by a pair tournament (as in
                    // cn_compute) merged into the row's (nm0, nm1), and the chunk's candidate isloc bits: the
                    // edges whose |lambda| equals the chunk minimum.  At the row end a chunk keeps them for the
                    // slots whose row minimum is its minimum (every edge of a tie: same eta, reading A13).
                    // Full chunks (warp-uniform) take a guard-free copy of the body.
                    auto chunk = [&](auto fullc) {
                        constexpr bool FC = decltype(fullc)::value;
                        float ax[C8][4], lo[4];
                        uint32_t iwc = 0u;
#pragma unroll
                        for (int u8 = 0; u8 < C8; u8++) {
                            const bool va = FC || p0 + u8 < d;
#pragma unroll
                            for (int v = 0; v < 4; v++) {
                                const float sj = comp(sv[u8], v);
                                float x;
                                if (FIRST) {
                                    x = __fadd_rn(sj, 0.0f);
                                } else {
                                    const float mag = (eb[u8] & (16u << v)) ? om1[v] : om0[v];
                                    x = __fadd_rn(__fsub_rn(sj, flip31(mag, eb[u8] << (31 - v))), 0.0f);
                                }
                                ax[u8][v] = va ? fabsf(x) : INF;
                                cw = __funnelshift_l(__float_as_uint(x), cw, 1);
                                if (EARLY) syn[v] ^= va ? __float_as_uint(sj) : 0u;
                            }
                        }
#pragma unroll
                        for (int v = 0; v < 4; v++) {
                            float l = fminf(ax[0][v], ax[1][v]), h = fmaxf(ax[0][v], ax[1][v]);
#pragma unroll
                            for (int u8 = 2; u8 < C8; u8 += 2) {
                                const float l2 = fminf(ax[u8][v], ax[u8 + 1][v]), h2 = fmaxf(ax[u8][v], ax[u8 + 1][v]);
                                h = fmin3f(h, h2, fmaxf(l, l2));
                                l = fminf(l, l2);
                            }
                            nm1[v] = fmin3f(nm1[v], h, fmaxf(nm0[v], l));
                            nm0[v] = fminf(nm0[v], l);
                            lo[v] = l;
                        }
#pragma unroll
                        for (int u8 = 0; u8 < C8; u8++)
#pragma unroll
                            for (int v = 0; v < 4; v++)
                                iwc = __funnelshift_l(__float_as_uint(__fsub_rn(lo[v], ax[u8][v])), iwc, 1);
#pragma unroll
                        for (int q = 0; q < (NWK > 0 ? NWK : 1); q++)
                            if (q == (p0 >> 3)) {
                                cls[q] = __brev(~iwc);  // bit 4u+v: |lambda| = chunk minimum
#pragma unroll
                                for (int v = 0; v < 4; v++) clo[q][v] = lo[v];
                            }
                        cw = __brev(cw);
                        if (!FC) cw &= (1u << (4 * (d - p0))) - 1u;
                    };
                    if (full) chunk(std::true_type{});
                    else chunk(std::false_type{});
                } else
#endif
                {
#if CNG_PAIR
#pragma unroll
                for (int u8 = 0; u8 < C8; u8 += 2) {  // edge pairs, as in cn_compute
                    const int p = p0 + u8;
                    const bool va = full || p < d, vb = full || p + 1 < d;
                    if (va) {
                        float xa[4], xb[4];
#pragma unroll
                        for (int v = 0; v < 4; v++) {
                            const float sa = comp(sv[u8], v), sb = comp(sv[u8 + 1], v);
                            if (FIRST) {
                                xa[v] = __fadd_rn(sa, 0.0f);
                                xb[v] = __fadd_rn(sb, 0.0f);
                            } else {
                                const float ma = (eb[u8] & (16u << v)) ? om1[v] : om0[v];
                                const float mb = (eb[u8 + 1] & (16u << v)) ? om1[v] : om0[v];
                                xa[v] = __fadd_rn(__fsub_rn(sa, flip31(ma, eb[u8] << (31 - v))), 0.0f);
                                xb[v] = __fadd_rn(__fsub_rn(sb, flip31(mb, eb[u8 + 1] << (31 - v))), 0.0f);
                            }
                            if (EARLY) syn[v] ^= __float_as_uint(sa) ^ (vb ? __float_as_uint(sb) : 0u);
                        }
#pragma unroll
                        for (int v = 0; v < 4; v++) cw = __funnelshift_l(__float_as_uint(xa[v]), cw, 1);
                        if (vb) {
#pragma unroll
                            for (int v = 0; v < 4; v++) cw = __funnelshift_l(__float_as_uint(xb[v]), cw, 1);
                        }
#pragma unroll
                        for (int v = 0; v < 4; v++) {
                            const float a = fabsf(xa[v]), b = vb ? fabsf(xb[v]) : INF;
                            const float sm = fminf(a, b), tm = fmaxf(a, b);
                            const int lp = b < a ? p + 1 : p;
                            const bool lt = sm < nm0[v];
                            nm1[v] = fmin3f(nm1[v], fmaxf(nm0[v], sm), tm);
                            nm0[v] = fminf(nm0[v], sm);
                            nloc[v] = lt ? lp : nloc[v];
                        }
                    }
                }
#else
#pragma unroll
                for (int u8 = 0; u8 < C8; u8++) {
                    const int p = p0 + u8;
                    if (full || p < d) {
#pragma unroll
                        for (int v = 0; v < 4; v++) {
                            const float sj = comp(sv[u8], v);
                            float x;
                            if (FIRST) {
                                x = __fadd_rn(sj, 0.0f);
                            } else {
                                const float mag = (eb[u8] & (16u << v)) ? om1[v] : om0[v];
                                x = __fadd_rn(__fsub_rn(sj, flip31(mag, eb[u8] << (31 - v))), 0.0f);
                            }
                            const float ax = fabsf(x);
                            const bool lt = ax < nm0[v];  // first strict minimum (A13)
                            nm1[v] = fminf(nm1[v], fmaxf(nm0[v], ax));
                            nm0[v] = fminf(nm0[v], ax);
                            nloc[v] = lt ? p : nloc[v];
                            if (EARLY) syn[v] ^= __float_as_uint(sj);
                            cw = __funnelshift_l(__float_as_uint(x), cw, 1);
                        }
                    }
                }
#endif
                const int pushed = full ? 32 : 4 * (d - p0);
                cw = pushed == 32 ? __brev(cw) : __brev(cw) >> (32 - pushed);  // bit 4u+v: edge p0+u, slot 4l+v
                }
                pf ^= cw;
                if (NWK > 0) {
#pragma unroll
                    for (int q = 0; q < (NWK > 0 ? NWK : 1); q++)
                        if (q == (p0 >> 3)) cws[q] = cw;
                } else {
                    const uint32_t ze = cw & 0x0f0f0f0fu, zo = (cw >> 4) & 0x0f0f0f0fu;
#pragma unroll
                    for (int u8 = 0; u8 < C8; u8++)
                        if (full || p0 + u8 < d)
                            Ri[REC_EDGE0 + 32 * (p0 + u8) + lane] = (unsigned char)(((u8 & 1) ? zo : ze) >> (8 * (u8 >> 1)));
                }
            }
            if (NWK > 0) {  // edge bytes with their isloc nibbles, chunk by chunk
#pragma unroll
                for (int q = 0; q < (NWK > 0 ? NWK : 1); q++) {
                    if (8 * q < d) {
                        uint32_t lm = 0;
#if CNG_TREE
#pragma unroll
                        for (int v = 0; v < 4; v++) lm |= clo[q][v] == nm0[v] ? (0x11111111u << v) : 0u;
                        lm &= cls[q];
#else
#pragma unroll
                        for (int v = 0; v < 4; v++) {
                            const int r = nloc[v] - 8 * q;
                            lm |= (r >= 0 && r < 8) ? (1u << (4 * r + v)) : 0u;
                        }
#endif
                        const uint32_t ze = (cws[q] & 0x0f0f0f0fu) | ((lm & 0x0f0f0f0fu) << 4);
                        const uint32_t zo = ((cws[q] >> 4) & 0x0f0f0f0fu) | (lm & 0xf0f0f0f0u);
#pragma unroll
                        for (int u8 = 0; u8 < C8; u8++)
                            if (8 * q + u8 < d)
                                Ri[REC_EDGE0 + 32 * (8 * q + u8) + lane] =
                                    (unsigned char)(((u8 & 1) ? zo : ze) >> (8 * (u8 >> 1)));
                    }
                }
            } else {  // isloc bits into the min0Location bytes of this lane (same thread wrote them: ordered)
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    unsigned char *bp = Ri + REC_EDGE0 + 32 * nloc[v] + lane;
                    *bp = (unsigned char)(*bp | (16u << v));
                }
            }
            // sign parity per slot (Obs. 2): XOR of bits v, v+4, ... of the chunk words, times (-1)^{d_i} (A1)
            uint32_t pw = pf ^ (pf >> 16);
            pw ^= pw >> 8;
            pw ^= pw >> 4;
            pw ^= ((uint32_t)(d & 1) & (uint32_t)(!literal)) ? 0xfu : 0u;
            const uint32_t sb[4] = {pw << 31, (pw << 30) & 0x80000000u, (pw << 29) & 0x80000000u,
                                    (pw << 28) & 0x80000000u};
            st4(reinterpret_cast<float *>(Ri) + 4 * lane,
                make_float4(__uint_as_float(__float_as_uint(nm0[0]) | sb[0]), __uint_as_float(__float_as_uint(nm0[1]) | sb[1]),
                            __uint_as_float(__float_as_uint(nm0[2]) | sb[2]), __uint_as_float(__float_as_uint(nm0[3]) | sb[3])));
            st4(reinterpret_cast<float *>(Ri) + 128 + 4 * lane,
                make_float4(__uint_as_float(__float_as_uint(nm1[0]) | sb[0]), __uint_as_float(__float_as_uint(nm1[1]) | sb[1]),
                            __uint_as_float(__float_as_uint(nm1[2]) | sb[2]), __uint_as_float(__float_as_uint(nm1[3]) | sb[3])));
            if (EARLY) {
                const uint32_t dp = (uint32_t)(d & 1);
#pragma unroll
                for (int v = 0; v < 4; v++) u[v] |= __ballot_sync(FULL_MASK, ((syn[v] >> 31) ^ dp) != 0u);
            }
        }
        if (EARLY) {
            if (lane == 0) {
#pragma unroll
                for (int v = 0; v < 4; v++)
                    if (u[v]) atomicOr(&s_u[v], u[v]);
            }
            cta_sync();
            if (threadIdx.x < 4 && s_u[threadIdx.x])
                atomicOr(w.unsat + ((size_t)(k & 1) * w.Tcap + t) * 4 + threadIdx.x, s_u[threadIdx.x]);
        }
    }
}

// ------------------------------------------------------------------------------------------------
// Check node with the row's loads staged by the TMA engine (cp.async.bulk, SASS UBLKCP): each warp owns
// a ring of CNB_R row buffers in shared memory; for a row, the lane of edge p issues one 512-byte bulk
// copy of s_j for the tile's 128 slots and lane 0 one copy of the row record (min0, min1, edge blocks),
// all completing on the buffer's mbarrier.  While a row is computed from shared memory, the next
// CNB_R - 1 rows are in flight, and no register holds a load across the latency.  Rows of degree <= 32.
// ------------------------------------------------------------------------------------------------
#ifndef CNB_W
#define CNB_W 4  // warps per CTA
#endif
#ifndef CNB_R
#define CNB_R 3  // row buffers per warp
#endif

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}

template <bool FIRST, bool EARLY, int NWK>
__global__ void __launch_bounds__(CNB_W * 32, 1)
    k_cn_bulk(Graph g, StreamState w, int k, int literal, const int *kdev, int slot_bytes) {
    if (kdev) k = *kdev;
    extern __shared__ __align__(128) unsigned char cnb_smem[];
    __shared__ __align__(8) uint64_t bars[CNB_W][CNB_R];
    __shared__ uint32_t s_u[4];
    __shared__ int s_item;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cnt = w.tcount[k & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        w.tcount[(k + 1) & 1] = 0;
        w.work[WK_BN] = 0;
        w.ctl[CT_NSRC] = 0;
        if (w.nlaunch) w.nlaunch[4] += (unsigned long long)cnt;
    }
    if (lane == 0) {
        for (int r = 0; r < CNB_R; r++) mbar_init(&bars[warp][r], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    unsigned char *ring = cnb_smem + (size_t)warp * CNB_R * slot_bytes;
    uint32_t phases = 0;  // bit r: parity of the next completion of buffer r
    const int m = g.m, n = g.n;
    const int nrb = (m + CN_ROWS - 1) / CN_ROWS;
    const int items = cnt * nrb;
    const float INF = __int_as_float(0x7f800000);
    for (;;) {
        if (EARLY && threadIdx.x < 4) s_u[threadIdx.x] = 0;
        const int it = next_item(w.work + WK_CN, s_item);
        if (it >= items) break;
        const int y = it / nrb, x = it - y * nrb;
        const int t = w.tlist[(size_t)(k & 1) * w.Tcap + y];
        const float *__restrict__ Sb = (FIRST ? w.r : w.s) + (size_t)t * n * TILE;
        unsigned char *RB = w.rst + (size_t)t * m * w.rs;
        const int i0 = x * CN_ROWS + warp, i1 = min(m, x * CN_ROWS + CN_ROWS);
        const int nr = i0 < i1 ? (i1 - i0 + CNB_W - 1) / CNB_W : 0;  // rows of this warp (<= 32)
        int ra = 0, rb = 0;
        if (lane < nr) {
            ra = __ldg(g.row_ptr + i0 + CNB_W * lane);
            rb = __ldg(g.row_ptr + i0 + CNB_W * lane + 1);
        }
        // issue the loads of the warp's row q into buffer q % CNB_R
        auto issue = [&](int q) {
            const int a = __shfl_sync(FULL_MASK, ra, q), d = __shfl_sync(FULL_MASK, rb, q) - a;
            const int r = q % CNB_R;
            unsigned char *buf = ring + (size_t)r * slot_bytes;
            const int cj = lane < d ? __ldg(g.col_idx + a + lane) : 0;
            if (lane == 0) {
                // the buffer was last read by this warp's generic-proxy loads: order them before the copies
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bars[warp][r], (uint32_t)(d * 512 + (FIRST ? 0 : REC_EDGE0 + 32 * d)));
            }
            __syncwarp();
            if (lane < d) bulk_g2s(buf + 512 * lane, Sb + (size_t)cj * TILE, 512u, &bars[warp][r]);
            if (!FIRST && lane == 0)
                bulk_g2s(buf + 512 * d, RB + (size_t)(i0 + CNB_W * q) * w.rs, (uint32_t)(REC_EDGE0 + 32 * d),
                         &bars[warp][r]);
        };
        for (int q = 0; q < CNB_R - 1 && q < nr; q++) issue(q);
        uint32_t u[4] = {0u, 0u, 0u, 0u};
        for (int q = 0; q < nr; q++) {
            if (q + CNB_R - 1 < nr) issue(q + CNB_R - 1);
            const int r = q % CNB_R;
            const int a = __shfl_sync(FULL_MASK, ra, q), d = __shfl_sync(FULL_MASK, rb, q) - a;
            (void)a;
            mbar_wait(&bars[warp][r], (phases >> r) & 1u);
            phases ^= 1u << r;
            const unsigned char *buf = ring + (size_t)r * slot_bytes;
            const unsigned char *rec = buf + 512 * d;  // the staged row record
            unsigned char *Ri = RB + (size_t)(i0 + CNB_W * q) * w.rs;
            float om0[4] = {0.f, 0.f, 0.f, 0.f}, om1[4] = {0.f, 0.f, 0.f, 0.f};
            if (!FIRST) {
                const float4 A = *reinterpret_cast<const float4 *>(rec + 16 * lane);
                const float4 B = *reinterpret_cast<const float4 *>(rec + 512 + 16 * lane);
                om0[0] = A.x; om0[1] = A.y; om0[2] = A.z; om0[3] = A.w;
                om1[0] = B.x; om1[1] = B.y; om1[2] = B.z; om1[3] = B.w;
            }
            float nm0[4] = {INF, INF, INF, INF}, nm1[4] = {INF, INF, INF, INF};
            int nloc[4] = {0, 0, 0, 0};
            uint32_t syn[4] = {0u, 0u, 0u, 0u}, pf = 0u;
            uint32_t cws[NWK];
#pragma unroll
            for (int c = 0; c < NWK; c++) {
                const int p0 = 8 * c;
                if (p0 >= d) break;
                const bool full = p0 + 8 <= d;
                uint32_t cw = 0;
#pragma unroll
                for (int u8 = 0; u8 < 8; u8++) {
                    const int p = p0 + u8;
                    if (full || p < d) {
                        const float4 sv = *reinterpret_cast<const float4 *>(buf + 512 * p + 16 * lane);
                        const uint32_t eb = FIRST ? 0u : rec[REC_EDGE0 + 32 * p + lane];
#pragma unroll
                        for (int v = 0; v < 4; v++) {
                            const float sj = comp(sv, v);
                            float xv;
                            if (FIRST) {
                                xv = __fadd_rn(sj, 0.0f);
                            } else {
                                const float mag = (eb & (16u << v)) ? om1[v] : om0[v];
                                xv = __fadd_rn(__fsub_rn(sj, flip31(mag, eb << (31 - v))), 0.0f);
                            }
                            const float ax = fabsf(xv);
                            const bool lt = ax < nm0[v];  // first strict minimum (A13)
                            nm1[v] = fminf(nm1[v], fmaxf(nm0[v], ax));
                            nm0[v] = fminf(nm0[v], ax);
                            nloc[v] = lt ? p : nloc[v];
                            if (EARLY) syn[v] ^= __float_as_uint(sj);
                            cw = __funnelshift_l(__float_as_uint(xv), cw, 1);
                        }
                    }
                }
                const int pushed = full ? 32 : 4 * (d - p0);
                cw = pushed == 32 ? __brev(cw) : __brev(cw) >> (32 - pushed);
                pf ^= cw;
                cws[c] = cw;
            }
#pragma unroll
            for (int c = 0; c < NWK; c++) {
                if (8 * c < d) {
                    uint32_t lm = 0;
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        const int rr = nloc[v] - 8 * c;
                        lm |= (rr >= 0 && rr < 8) ? (1u << (4 * rr + v)) : 0u;
                    }
                    const uint32_t ze = (cws[c] & 0x0f0f0f0fu) | ((lm & 0x0f0f0f0fu) << 4);
                    const uint32_t zo = ((cws[c] >> 4) & 0x0f0f0f0fu) | (lm & 0xf0f0f0f0u);
#pragma unroll
                    for (int u8 = 0; u8 < 8; u8++)
                        if (8 * c + u8 < d)
                            Ri[REC_EDGE0 + 32 * (8 * c + u8) + lane] = (unsigned char)(((u8 & 1) ? zo : ze) >> (8 * (u8 >> 1)));
                }
            }
            uint32_t pw = pf ^ (pf >> 16);
            pw ^= pw >> 8;
            pw ^= pw >> 4;
            pw ^= ((uint32_t)(d & 1) & (uint32_t)(!literal)) ? 0xfu : 0u;
            const uint32_t sb[4] = {pw << 31, (pw << 30) & 0x80000000u, (pw << 29) & 0x80000000u,
                                    (pw << 28) & 0x80000000u};
            st4(reinterpret_cast<float *>(Ri) + 4 * lane,
                make_float4(__uint_as_float(__float_as_uint(nm0[0]) | sb[0]), __uint_as_float(__float_as_uint(nm0[1]) | sb[1]),
                            __uint_as_float(__float_as_uint(nm0[2]) | sb[2]), __uint_as_float(__float_as_uint(nm0[3]) | sb[3])));
            st4(reinterpret_cast<float *>(Ri) + 128 + 4 * lane,
                make_float4(__uint_as_float(__float_as_uint(nm1[0]) | sb[0]), __uint_as_float(__float_as_uint(nm1[1]) | sb[1]),
                            __uint_as_float(__float_as_uint(nm1[2]) | sb[2]), __uint_as_float(__float_as_uint(nm1[3]) | sb[3])));
            if (EARLY) {
                const uint32_t dp = (uint32_t)(d & 1);
#pragma unroll
                for (int v = 0; v < 4; v++) u[v] |= __ballot_sync(FULL_MASK, ((syn[v] >> 31) ^ dp) != 0u);
            }
            __syncwarp();  // every lane has read the buffer before it is refilled
        }
        if (EARLY) {
            if (lane == 0) {
#pragma unroll
                for (int v = 0; v < 4; v++)
                    if (u[v]) atomicOr(&s_u[v], u[v]);
            }
            cta_sync();
            if (threadIdx.x < 4 && s_u[threadIdx.x])
                atomicOr(w.unsat + ((size_t)(k & 1) * w.Tcap + t) * 4 + threadIdx.x, s_u[threadIdx.x]);
        }
    }
}

// ------------------------------------------------------------------------------------------------
// a5/a6: bit-node sweep of loop body k; stops frames whose b^(k-1) satisfied every check.
// Item = 16 columns of one tile; a warp walks each of its columns' edges one at a time (broadcast edge
// record, then three loads: min0, min1 -- 512 B each per warp -- and the lane's edge byte), with few
// registers and 48 warps per SM to keep the loads in flight.
// The item with block 0 of a tile does the tile's bookkeeping: newly stopped frames (k, isCodeword),
// and the tile goes to the list of body k+1 -- or, when fewer than half of its slots still run and
// at least two bodies remain, to the compaction sources.
// ------------------------------------------------------------------------------------------------
// How the bit node gathers (A/B, 8192 frames at the lowest Eb/N0, every frame running, early stop off;
// C3 / C4 ms per 20 / 10 bodies):
//   BN_V8 = 1  256-bit accesses, half-warps on separate columns, 8 slots per lane, 12 CTAs x 128 threads:
//              12.74 / 27.39 (C6 3.27 against 3.96);
//   BN_V8 = 0  float4 accesses, 4 slots per lane, per-edge offset records (Graph::bn_off, 32-byte units;
//              one IMAD.WIDE per address): 14.57 / 30.82 (round-1 {e, i, p} records: 15.27 / 32.15).
// Measured and removed: the next column's edge list prefetched into lanes (slower: fewer warps or
// spills), the next edge's record loaded one edge ahead (equal), two edges per step (equal), loads of
// 2-5 edges together (0-15 % slower), min1 loaded only where the edge is a min0Location (25 % slower),
// row state staged through shared memory with cp.async 3-8 edges deep per warp (40-55 % slower),
// 256-bit accesses at 8 / 10 / 14 / 16 CTAs per SM (slower than 12).
#ifndef BN_V8
#define BN_V8 1
#endif
#ifndef COMPACT_PCT
#define COMPACT_PCT 50  // a tile with fewer than this percentage of its slots running becomes a compaction source
#endif

#ifndef BN_DYN
#define BN_DYN 1  // items from the work counter (keeps the tiles in flight together for L2 reuse)
#endif

#if !BN_V8
// s of one column for this lane's 4 slots: new values for the running frames, r for frames stopped at
// the pre-check (body 1), untouched for frozen frames; zeros kept as -0 (A12)
__device__ __forceinline__ void bn_store(float *o, const float (&acc)[4], float4 rv, unsigned mine, int k,
                                         uint64_t pf) {
    const float n0 = zneg(acc[0] + rv.x), n1 = zneg(acc[1] + rv.y), n2 = zneg(acc[2] + rv.z),
                n3 = zneg(acc[3] + rv.w);
    if (mine == 0xFu) {
        sth4<1, L2H_BN>(o, make_float4(n0, n1, n2, n3), pf);
    } else if (k == 1) {  // body 1: frames that stopped at the pre-check keep s = r
        st4(o, make_float4((mine & 1u) ? n0 : rv.x, (mine & 2u) ? n1 : rv.y, (mine & 4u) ? n2 : rv.z,
                           (mine & 8u) ? n3 : rv.w));
    } else if (mine) {  // frozen frames keep their s
        if (mine & 1u) o[0] = n0;
        if (mine & 2u) o[1] = n1;
        if (mine & 4u) o[2] = n2;
        if (mine & 8u) o[3] = n3;
    }
}
#endif


template <bool EARLY>
__global__ void __launch_bounds__(BN_T, BN_MINB)
    k_bn(Graph g, StreamState w, int k, int L, const int *kdev, int check_every, int compact) {
    if (kdev) k = *kdev;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int Tc = w.Tcap;
    __shared__ int s_item;
    const int cnt = w.tcount[k & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        w.work[WK_CN] = 0;  // next check-node sweep
        w.work[WK_MOVE] = 0;
        w.work[WK_SYN] = 0;
        if (w.nlaunch) w.nlaunch[5] += (unsigned long long)cnt;  // tile-bodies swept by the bit node
    }
    const int m = g.m, n = g.n;
    const int ncb = (n + BN_COLS - 1) / BN_COLS;
    const int items = cnt * ncb;
    const bool compact_ok = EARLY && compact && k + 2 <= L;
    const uint64_t pf = (L2H_BN & 1) ? pol_first() : 0, pl = (L2H_BN & 2) ? pol_last() : 0;
    for (int it0 = blockIdx.x;; it0 += gridDim.x) {
        const int it = BN_DYN ? next_item(w.work + WK_BN, s_item) : it0;
        if (it >= items) break;
        const int y = it / ncb, x = it - y * ncb;
        const int t = w.tlist[(size_t)(k & 1) * Tc + y];
        uint4 act = make_uint4(FULL_MASK, FULL_MASK, FULL_MASK, FULL_MASK);
        if (EARLY) {
            // the syndrome of k_cn(k) tests b^(k-1); it may stop frames only at a check point (k-1) % T == 0
            const bool check = ((k - 1) % check_every) == 0;
            const uint4 ua = check ? ldu4(w.unsat + ((size_t)(k & 1) * Tc + t) * 4)
                                   : make_uint4(FULL_MASK, FULL_MASK, FULL_MASK, FULL_MASK);
            const uint4 dw = ldu4(w.done + (size_t)t * 4);
            const uint4 newly = make_uint4(~ua.x & ~dw.x, ~ua.y & ~dw.y, ~ua.z & ~dw.z, ~ua.w & ~dw.w);
            act = make_uint4(ua.x & ~dw.x, ua.y & ~dw.y, ua.z & ~dw.z, ua.w & ~dw.w);
            if (x == 0) {  // the tile's bookkeeping item (uniform in the CTA)
                // every thread has read `done` before it is rewritten (other items of the tile may see either
                // value: act is the same for both, since newly and ua are disjoint)
                cta_sync();
                const int tid = threadIdx.x;
                if (tid < 4) {
                    w.done[(size_t)t * 4 + tid] = comp(dw, tid) | comp(newly, tid);
                    w.unsat[((size_t)((k + 1) & 1) * Tc + t) * 4 + tid] = 0;  // buffer of body k+1
                }
                if (tid < TILE && ((comp(newly, tid & 3) >> (tid >> 2)) & 1u)) {
                    const int f = w.fid[(size_t)t * TILE + tid];
                    w.iters[f] = k - 1;  // stopped after k-1 bodies
                    w.conv[f] = 1;
                }
                if (tid == 0) {
                    const int run = __popc(act.x) + __popc(act.y) + __popc(act.z) + __popc(act.w);
                    if (run > 0 && compact_ok && 100 * run < COMPACT_PCT * TILE) {  // compaction source
                        const int pos = atomicAdd(w.ctl + CT_NSRC, 1);
                        w.csrc[pos] = t;
                        w.ccnt[pos] = run;
                    } else if (run > 0) {  // the tile still runs in body k+1
                        const int pos = atomicAdd(w.tcount + ((k + 1) & 1), 1);
                        w.tlist[(size_t)((k + 1) & 1) * Tc + pos] = t;
                    }
                }
            }
            if (k > 1 && (act.x | act.y | act.z | act.w) == 0) continue;
        } else if (x == 0 && threadIdx.x == 0) {
            const int pos = atomicAdd(w.tcount + ((k + 1) & 1), 1);
            w.tlist[(size_t)((k + 1) & 1) * Tc + pos] = t;
        }
        const unsigned char *RB = w.rst + (size_t)t * m * w.rs;
#if !BN_V8
        const unsigned mine = ((act.x >> lane) & 1u) | (((act.y >> lane) & 1u) << 1) | (((act.z >> lane) & 1u) << 2) |
                              (((act.w >> lane) & 1u) << 3);
        const size_t tb = (size_t)t * n * TILE + 4 * lane;  // r and s of the tile (one offset, two bases)
#endif
        const int j1 = min(n, x * BN_COLS + BN_COLS);
#if BN_V8
        // 256-bit accesses: half-warp h (lanes 16h..16h+15) sweeps its own columns, half-lane hl owns the 8
        // slots 8hl..8hl+7 (32 contiguous bytes of min0, of min1, of r and of s; its two edge-block bytes in
        // one 16-bit load).  One warp instruction moves two edges' worth of row state for 128 slots, so a
        // warp keeps twice the bytes in flight with half the load instructions per edge.
        {
            const int hw = (warp << 1) | (lane >> 4), hl = lane & 15;
            // slot 8hl + v of the tile = old lane 2hl + (v >> 2), component v & 3: bit v of mine8
            const unsigned mine8 = ((act.x >> (2 * hl)) & 1u) | (((act.y >> (2 * hl)) & 1u) << 1) |
                                   (((act.z >> (2 * hl)) & 1u) << 2) | (((act.w >> (2 * hl)) & 1u) << 3) |
                                   (((act.x >> (2 * hl + 1)) & 1u) << 4) | (((act.y >> (2 * hl + 1)) & 1u) << 5) |
                                   (((act.z >> (2 * hl + 1)) & 1u) << 6) | (((act.w >> (2 * hl + 1)) & 1u) << 7);
            const unsigned char *RBm = RB + 32 * hl, *RBb = RB + 2 * hl;
            const size_t tb8 = (size_t)t * n * TILE + 8 * hl;
            constexpr int NHW = BN_T / 16;  // half-warps per CTA
            for (int jb = x * BN_COLS; jb < j1; jb += NHW) {  // warp-uniform trip count
                const int j = jb + hw;
                const bool colok = j < j1;
                const int c0 = colok ? __ldg(g.col_ptr + j) : 0, dv = colok ? __ldg(g.col_ptr + j + 1) - c0 : 0;
                float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                const int2 *op = g.bn_off + c0;  // ascending i (A14)
#pragma unroll 1
                for (int q = 0; q < dv; q++, op++) {
                    const int2 o = __ldg(op);
                    const float *Rm = reinterpret_cast<const float *>(RBm + ((size_t)(unsigned)o.x << 5));
                    const f8 m0 = ld8h<L2H_BN>(Rm, pl), m1 = ld8h<L2H_BN>(Rm + 128, pl);
                    const uint32_t b = *reinterpret_cast<const uint16_t *>(RBb + ((size_t)(unsigned)o.y << 5));
#pragma unroll
                    for (int v = 0; v < 8; v++) {
                        const int sb = v < 4 ? v : v + 4;  // sign bit of slot v; its isloc bit is sb + 4
                        const float mag = (b & (16u << sb)) ? m1.v[v] : m0.v[v];  // Obs. 1
                        acc[v] = acc[v] + flip31(mag, b << (31 - sb));
                    }
                }
                if (colok) {
                    float *o8 = w.s + tb8 + (size_t)j * TILE;
                    const f8 rv = ld8h<L2H_BN>(w.r + tb8 + (size_t)j * TILE, pf);
                    f8 nv;
#pragma unroll
                    for (int v = 0; v < 8; v++) nv.v[v] = zneg(acc[v] + rv.v[v]);  // zeros of s kept as -0 (A12)
                    if (mine8 == 0xFFu) {
                        st8h<L2H_BN>(o8, nv, pf);
                    } else if (k == 1) {  // body 1: frames that stopped at the pre-check keep s = r
#pragma unroll
                        for (int v = 0; v < 8; v++) nv.v[v] = ((mine8 >> v) & 1u) ? nv.v[v] : rv.v[v];
                        st8h<0>(o8, nv, pf);
                    } else if (mine8) {  // frozen frames keep their s
#pragma unroll
                        for (int v = 0; v < 8; v++)
                            if ((mine8 >> v) & 1u) o8[v] = nv.v[v];
                    }
                }
            }
        }
#else  // float4 accesses, per-edge offset records
        // per-edge offset records (Graph::bn_off, 32-byte units): one IMAD.WIDE per gather address, the
        // record pointer advanced by 8 bytes per edge
        const unsigned char *RBm = RB + 16 * lane, *RBb = RB + lane;
        for (int j = x * BN_COLS + warp; j < j1; j += BN_T / 32) {
            const int c0 = __ldg(g.col_ptr + j), dv = __ldg(g.col_ptr + j + 1) - c0;
            const float4 rv = ldh4<1, L2H_BN>(w.r + tb + (size_t)j * TILE, pf);
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            const int2 *op = g.bn_off + c0;  // ascending i (A14)
            int q = 0;
#pragma unroll 1
            for (; q < dv; q++, op++) {
                const int2 o = __ldg(op);
                const float *Rm = reinterpret_cast<const float *>(RBm + ((size_t)(unsigned)o.x << 5));
                const float4 m0 = ldh4<2, L2H_BN>(Rm, pl);
                const float4 m1 = ldh4<2, L2H_BN>(Rm + 128, pl);
                const uint32_t b = RBb[(size_t)(unsigned)o.y << 5];
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    const float mag = (b & (16u << v)) ? comp(m1, v) : comp(m0, v);  // Obs. 1
                    acc[v] = acc[v] + flip31(mag, b << (31 - v));
                }
            }
#endif
#if !BN_V8
            bn_store(w.s + tb + (size_t)j * TILE, acc, rv, mine, k, pf);
        }
#endif
    }
}

__global__ void k_bn_offsets(const int4 *__restrict__ bn_edge, int E, int rs32, int2 *__restrict__ out) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= E) return;
    const int4 ed = bn_edge[q];  // {e, i, p, d_i & 1}
    out[q] = make_int2(ed.y * rs32, ed.y * rs32 + REC_EDGE0 / 32 + ed.z);
}

// ------------------------------------------------------------------------------------------------
// f1: compaction of the sources the bit node of body k collected (tiles with fewer than 64 running
// frames).  Plan (one CTA): the running frames of the sources, in (source, slot) order, get the
// slots of ceil(R/128) fresh tiles at the end of the workspace; the fresh tiles join the list of body
// k+1, the sources are retired (their stopped frames stay in place for the stage-out).  If that would
// not save a tile (or the workspace is full), the sources simply stay in the list.
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_compact_plan(StreamState w, int k, const int *kdev) {
    if (kdev) k = *kdev;
    __shared__ int s_part[1024];
    __shared__ int s_tot;
    const int tid = threadIdx.x, NT = blockDim.x, Tc = w.Tcap;
    const int nsrc = w.ctl[CT_NSRC];
    if (nsrc == 0) {
        if (tid == 0) w.ctl[CT_NDST] = 0;
        return;
    }
    // exclusive scan of the running counts (contiguous ranges per thread)
    const int per = (nsrc + NT - 1) / NT, a = min(nsrc, tid * per), b = min(nsrc, a + per);
    int sum = 0;
    for (int q = a; q < b; q++) sum += w.ccnt[q];
    s_part[tid] = sum;
    cta_sync();
    if (tid == 0) {
        int run = 0;
        for (int q = 0; q < NT; q++) {
            const int v = s_part[q];
            s_part[q] = run;
            run += v;
        }
        s_tot = run;
    }
    cta_sync();
    const int R = s_tot, ndst = (R + TILE - 1) / TILE, base = w.ctl[CT_TNEXT];
    const int nxt = (k + 1) & 1;
    if (ndst >= nsrc || base + ndst > Tc) {  // nothing to gain (or no room): the sources keep running
        if (tid == 0) w.ctl[CT_NDST] = 0;
        for (int q = tid; q < nsrc; q += NT) {
            const int pos = atomicAdd(w.tcount + nxt, 1);
            w.tlist[(size_t)nxt * Tc + pos] = w.csrc[q];
        }
        return;
    }
    int run = s_part[tid];
    for (int q = a; q < b; q++) {
        const int t = w.csrc[q];
        const uint4 dw = ldu4(w.done + (size_t)t * 4);
        for (int sl = 0; sl < TILE; sl++) {
            if ((comp(dw, sl & 3) >> (sl >> 2)) & 1u) continue;  // stopped (or padding): stays
            const int dt = run >> 7, ds = run & 127;
            run++;
            w.cmap[(size_t)dt * TILE + ds] = (t << 7) | sl;
            w.fid[(size_t)(base + dt) * TILE + ds] = w.fid[(size_t)t * TILE + sl];
            w.fid[(size_t)t * TILE + sl] = -1;  // moved: its outputs come from the fresh tile
        }
        w.done[(size_t)t * 4 + 0] = FULL_MASK;
        w.done[(size_t)t * 4 + 1] = FULL_MASK;
        w.done[(size_t)t * 4 + 2] = FULL_MASK;
        w.done[(size_t)t * 4 + 3] = FULL_MASK;
    }
    // fresh tiles: padding slots past R in the last one
    for (int q = tid; q < ndst * TILE; q += NT) {
        if (q >= R) {
            w.cmap[q] = -1;
            w.fid[(size_t)base * TILE + q] = -1;
        }
    }
    for (int dt = tid; dt < ndst; dt += NT) {
        const int T2 = base + dt;
        for (int v = 0; v < 4; v++) {
            uint32_t pad = 0;
            for (int l = 0; l < 32; l++)
                if (dt * TILE + 4 * l + v >= R) pad |= 1u << l;
            w.done[(size_t)T2 * 4 + v] = pad;
            w.unsat[(size_t)T2 * 4 + v] = 0;
            w.unsat[((size_t)Tc + T2) * 4 + v] = 0;
        }
        const int pos = atomicAdd(w.tcount + nxt, 1);
        w.tlist[(size_t)nxt * Tc + pos] = T2;
    }
    if (tid == 0) {
        w.ctl[CT_NDST] = ndst;
        w.ctl[CT_DBASE] = base;
        w.ctl[CT_TNEXT] = base + ndst;
        if (w.nlaunch) {  // handle counters: [1] frames moved, [2] compactions, [3] source tiles retired
            w.nlaunch[1] += (unsigned long long)R;
            w.nlaunch[2] += 1;
            w.nlaunch[3] += (unsigned long long)nsrc;
        }
    }
}

// Move (persistent): item = (fresh tile, 8 columns) -> s and r; or (fresh tile, 8 rows) -> min0, min1 and
// the edge bytes.  Lane l assembles slots 4l..4l+3 from their sources (scalar loads that hit the few
// source segments the tile draws from) and writes them with one 16-byte store / one byte per edge.
constexpr int MV_T = 256;

__global__ void __launch_bounds__(MV_T) k_compact_move(Graph g, StreamState w) {
    __shared__ int s_map[TILE];
    __shared__ int s_item;
    const int ndst = w.ctl[CT_NDST];
    if (ndst == 0) return;
    const int base = w.ctl[CT_DBASE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int m = g.m, n = g.n;
    const int nc = (n + 7) / 8, nrw = (m + 7) / 8, per = nc + nrw;
    const int items = ndst * per;
    for (;;) {
        const int it = next_item(w.work + WK_MOVE, s_item);
        if (it >= items) break;
        const int y = it / per, x = it - y * per;
        if (threadIdx.x < TILE) s_map[threadIdx.x] = w.cmap[(size_t)y * TILE + threadIdx.x];
        cta_sync();
        const int T2 = base + y;
        int src[4];
#pragma unroll
        for (int v = 0; v < 4; v++) src[v] = s_map[4 * lane + v];
        if (x < nc) {
            const int j = x * 8 + warp;
            if (j < n) {
                float sv[4], rv[4];
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    if (src[v] >= 0) {
                        const size_t o = ((size_t)(src[v] >> 7) * n + j) * TILE + (src[v] & 127);
                        sv[v] = w.s[o];
                        rv[v] = w.r[o];
                    } else {
                        sv[v] = rv[v] = -1.0f;
                    }
                }
                const size_t o = ((size_t)T2 * n + j) * TILE + 4 * lane;
                st4(w.s + o, make_float4(sv[0], sv[1], sv[2], sv[3]));
                st4(w.r + o, make_float4(rv[0], rv[1], rv[2], rv[3]));
            }
        } else {
            const int i = (x - nc) * 8 + warp;
            if (i < m) {
                const int d = __ldg(g.row_ptr + i + 1) - __ldg(g.row_ptr + i);
                float a0[4], a1[4];
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    if (src[v] >= 0) {
                        const float *Rs = reinterpret_cast<const float *>(w.rst + ((size_t)(src[v] >> 7) * m + i) * w.rs);
                        a0[v] = Rs[src[v] & 127];
                        a1[v] = Rs[128 + (src[v] & 127)];
                    } else {
                        a0[v] = a1[v] = 0.f;
                    }
                }
                unsigned char *Rd = w.rst + ((size_t)T2 * m + i) * w.rs;
                st4(reinterpret_cast<float *>(Rd) + 4 * lane, make_float4(a0[0], a0[1], a0[2], a0[3]));
                st4(reinterpret_cast<float *>(Rd) + 128 + 4 * lane, make_float4(a1[0], a1[1], a1[2], a1[3]));
                for (int p = 0; p < d; p++) {
                    uint32_t byte = 0;
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        if (src[v] >= 0) {
                            const int sq = src[v] & 127;
                            const uint32_t sb =
                                w.rst[((size_t)(src[v] >> 7) * m + i) * w.rs + REC_EDGE0 + 32 * p + (sq >> 2)];
                            byte |= ((sb >> (sq & 3)) & 1u) << v;             // sign
                            byte |= ((sb >> (4 + (sq & 3))) & 1u) << (4 + v);  // isloc
                        }
                    }
                    Rd[REC_EDGE0 + 32 * p + lane] = (unsigned char)byte;
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------------------
// a6: syndrome of b^(L) (the test after the last body), into unsat[slot], over the tiles still running.
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(CTA) k_syndrome(Graph g, StreamState w, int slot, const float *__restrict__ sfin) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t s_u[4];
    __shared__ int s_item;
    const int cnt = w.tcount[slot];  // tiles still running after the last body
    const int nrb = (g.m + CN_ROWS - 1) / CN_ROWS;
    const int items = cnt * nrb;
    for (;;) {
        if (threadIdx.x < 4) s_u[threadIdx.x] = 0;
        const int it = next_item(w.work + WK_SYN, s_item);
        if (it >= items) break;
        const int y = it / nrb, x = it - y * nrb;
        const int t = w.tlist[(size_t)slot * w.Tcap + y];
        const size_t tn = (size_t)t * g.n;
        const int i0 = x * CN_ROWS, i1 = min(g.m, i0 + CN_ROWS);
        uint32_t u[4] = {0, 0, 0, 0};
        for (int i = i0 + warp; i < i1; i += CTA / 32) {
            const int a = __ldg(g.row_ptr + i), d = __ldg(g.row_ptr + i + 1) - a;
            unsigned syn = 0;
            for (int p = 0; p < d; p++) {
                const int j = __ldg(g.col_idx + a + p);
                const float4 sv = ld4(sfin + (tn + j) * TILE + 4 * lane);
                syn ^= (unsigned)(sv.x > 0.f) | ((unsigned)(sv.y > 0.f) << 1) | ((unsigned)(sv.z > 0.f) << 2) |
                       ((unsigned)(sv.w > 0.f) << 3);
            }
#pragma unroll
            for (int v = 0; v < 4; v++) u[v] |= __ballot_sync(FULL_MASK, (syn >> v) & 1u);
        }
        if (lane == 0)
#pragma unroll
            for (int v = 0; v < 4; v++)
                if (u[v]) atomicOr(&s_u[v], u[v]);
        cta_sync();
        if (threadIdx.x < 4 && s_u[threadIdx.x])
            atomicOr(w.unsat + ((size_t)slot * w.Tcap + t) * 4 + threadIdx.x, s_u[threadIdx.x]);
    }
}

// ------------------------------------------------------------------------------------------------
// a7: stage-out.  For every tile ever used and every slot holding a frame (fid >= 0): posterior
// [F][n] = s, bits = slice(s) (transposed through shared memory: 128-byte rows per frame), the
// per-frame bit errors and near-zero flag; block 0 of a tile also settles the frames that ran all L
// bodies (k = L, isCodeword = the final syndrome).
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(CTA) k_finalize(StreamState w, int n, int L, int final_slot,
                                                  const float *__restrict__ sfin, float *__restrict__ post,
                                                  uint8_t *__restrict__ bits) {
    __shared__ float ts[32][TILE + 1];
    __shared__ int s_fid[TILE];
    const int t = blockIdx.y;
    if (t >= w.ctl[CT_TNEXT]) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < TILE) {
        const int q = threadIdx.x, f = w.fid[(size_t)t * TILE + q];
        s_fid[q] = f;
        if (blockIdx.x == 0 && f >= 0) {
            const uint32_t dn = w.done[(size_t)t * 4 + (q & 3)];
            if (!((dn >> (q >> 2)) & 1u)) {  // still running after body L
                w.iters[f] = L;
                w.conv[f] = !((w.unsat[((size_t)final_slot * w.Tcap + t) * 4 + (q & 3)] >> (q >> 2)) & 1u);
            }
        }
    }
    cta_sync();
    int be_acc = 0;  // lane q < 16 of warp w: slot w + 8q
    bool nz_acc = false;
    for (int sb = 0; sb < SI_SUB; sb++) {
        const int j0 = (blockIdx.x * SI_SUB + sb) * 32;
        if (j0 >= n) break;
        for (int jl = warp; jl < 32; jl += CTA / 32) {
            const int j = j0 + jl;
            if (j >= n) break;
            const size_t base = ((size_t)t * n + j) * TILE;
#pragma unroll
            for (int q = 0; q < 4; q++) ts[jl][lane + 32 * q] = sfin[base + lane + 32 * q];
        }
        cta_sync();
        const int j = j0 + lane;
        const bool jv = j < n;
#pragma unroll 4
        for (int q = 0; q < TILE / (CTA / 32); q++) {
            const int sl = warp + (CTA / 32) * q;
            const int f = s_fid[sl];
            if (f < 0) continue;  // warp-uniform
            const float sv = ts[lane][sl];
            const bool b = jv && sv > 0.f;  // Eq. slice
            if (jv) {
                if (post) post[(int64_t)f * n + j] = sv;
                if (bits) bits[(int64_t)f * n + j] = (uint8_t)b;
            }
            const int be = __popc(__ballot_sync(FULL_MASK, b));
            const bool nz = __any_sync(FULL_MASK, jv && fabsf(sv) <= 1e-4f);
            if (lane == q) {
                be_acc += be;
                nz_acc = nz_acc || nz;
            }
        }
        cta_sync();  // the next sub-block overwrites ts
    }
    if (lane < TILE / (CTA / 32)) {
        const int f = s_fid[warp + (CTA / 32) * lane];
        if (f >= 0) {
            if (be_acc) atomicAdd(w.fbe + f, be_acc);
            if (nz_acc) w.fnz[f] = 1;
        }
    }
}

// per-frame k, isCodeword and the 8 accumulated counters
__global__ void __launch_bounds__(CTA) k_frame_stats(StreamState w, int64_t frames, int32_t *__restrict__ iters_out,
                                                     uint8_t *__restrict__ conv_out,
                                                     unsigned long long *__restrict__ stats) {
    __shared__ unsigned long long s_acc[8];
    if (threadIdx.x < 8) s_acc[threadIdx.x] = 0;
    cta_sync();
    const int64_t f = blockIdx.x * (int64_t)CTA + threadIdx.x;
    unsigned long long c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (f < frames) {
        const int it = w.iters[f], conv = w.conv[f];
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
            for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL_MASK, x, o);
            if ((threadIdx.x & 31) == 0 && x) atomicAdd(&s_acc[q], x);
        }
        cta_sync();
        if (threadIdx.x < 8 && s_acc[threadIdx.x]) atomicAdd(stats + threadIdx.x, s_acc[threadIdx.x]);
    }
}

// Graph-driven loop control (CUDA conditional WHILE node): body k runs while k <= L and some tile
// still has a running frame.  On an early end, the list the final syndrome pass reads is emptied.
__global__ void k_loop_pre(StreamState w, int L, cudaGraphConditionalHandle h) {
    const int k = 2;
    const bool run = k <= L && w.tcount[k & 1] > 0;
    *w.kdev = k;
    if (run && w.nlaunch) *w.nlaunch += BODY_LAUNCHES;
    if (!run) w.tcount[(L + 1) & 1] = 0;
    cudaGraphSetConditional(h, run ? 1u : 0u);
}

__global__ void k_loop_step(StreamState w, int L, cudaGraphConditionalHandle h) {
    const int k = *w.kdev + 1;
    const bool run = k <= L && w.tcount[k & 1] > 0;
    *w.kdev = k;
    if (run && w.nlaunch) *w.nlaunch += BODY_LAUNCHES;
    if (!run && k <= L) w.tcount[(L + 1) & 1] = 0;
    cudaGraphSetConditional(h, run ? 1u : 0u);
}

inline dim3 grid2(int64_t x, int y) { return dim3((unsigned)std::max<int64_t>(1, x), (unsigned)y); }

// shared memory of one CTA of the bulk-staged check node (CNB_W warps x CNB_R row buffers), 0 if the
// rows are too long for it
size_t cn_bulk_smem(int dmax) {
    if (dmax > 32) return 0;
    const int ecap = dmax <= 8 ? 8 : dmax <= 16 ? 16 : 32;
    const size_t slot = ((size_t)512 * ecap + REC_EDGE0 + 32 * ecap + 127) / 128 * 128;
    return slot * CNB_W * CNB_R;
}

template <bool F, bool EA, int NWK>
void cnb_launch(const Graph &g, const StreamState &w, int k, int lit, const StreamLaunch &cfg, cudaStream_t st,
                const int *kdev) {
    const size_t smem = cn_bulk_smem(g.dmax);
    const int slot = (int)(smem / (CNB_W * CNB_R));
    int per_sm = cfg.smem_per_sm > 0 ? (int)(cfg.smem_per_sm / (smem + 2048)) : 1;
    per_sm = std::max(1, std::min(per_sm, 8));
    cudaFuncSetAttribute(k_cn_bulk<F, EA, NWK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_cn_bulk<F, EA, NWK><<<cfg.sms * per_sm, CNB_W * 32, smem, st>>>(g, w, k, lit, kdev, slot);
}

template <bool F, bool EA>
void cn_launch(const Graph &g, const StreamState &w, int k, int lit, const StreamLaunch &cfg, cudaStream_t st,
               const int *kdev) {
    const dim3 grid(cfg.sms * CN_MINB), gridg(cfg.sms * CNG_MINB);
    if (cfg.cn_bulk && g.dmax <= 32) {
        if (g.dmax <= 8) cnb_launch<F, EA, 1>(g, w, k, lit, cfg, st, kdev);
        else if (g.dmax <= 16) cnb_launch<F, EA, 2>(g, w, k, lit, cfg, st, kdev);
        else cnb_launch<F, EA, 4>(g, w, k, lit, cfg, st, kdev);
    } else if (!cfg.cn_generic && g.dmax <= 8) {
        if (g.dmax <= 4) k_cn<4, F, EA><<<grid, CN_T, 0, st>>>(g, w, k, lit, kdev);
        else if (g.dmax <= 6) k_cn<6, F, EA><<<grid, CN_T, 0, st>>>(g, w, k, lit, kdev);
        else if (g.dmax == 7) k_cn<7, F, EA><<<grid, CN_T, 0, st>>>(g, w, k, lit, kdev);
        else k_cn<8, F, EA><<<grid, CN_T, 0, st>>>(g, w, k, lit, kdev);
    } else if (g.dmax <= 16) {
        k_cn_generic<F, EA, 2><<<gridg, CN_T, 0, st>>>(g, w, k, lit, kdev);
    } else if (g.dmax <= 32) {
        k_cn_generic<F, EA, 4><<<gridg, CN_T, 0, st>>>(g, w, k, lit, kdev);
    } else {
        k_cn_generic<F, EA, 0><<<gridg, CN_T, 0, st>>>(g, w, k, lit, kdev);
    }
}

}  // namespace

int edge_capacity(int dmax, bool generic) {
    if (!generic && dmax <= 8) return dmax <= 4 ? 4 : dmax <= 6 ? 6 : dmax == 7 ? 7 : 8;
    return (dmax + 7) / 8 * 8;
}

int launch_bn_offsets(const Graph &g, int rs, int2 *out, cudaStream_t st) {
    k_bn_offsets<<<(g.E + 255) / 256, 256, 0, st>>>(g.bn_edge, g.E, rs / 32, out);
    return 1;
}

int launch_stage_in(const Graph &g, const StreamState &w, const float *llr, int64_t frames, cudaStream_t st) {
    cudaMemsetAsync(w.fcnt, 0, sizeof(int) * 3 * (size_t)w.T * TILE, st);  // fbe, fraw, fnz
    k_stage_in<<<grid2((g.n + 32 * SI_SUB - 1) / (32 * SI_SUB), w.T), CTA, 0, st>>>(llr, frames, g.n, w);
    return 1;
}

int launch_check_node(const Graph &g, const StreamState &w, int k, bool first, bool early, bool literal,
                      const StreamLaunch &cfg, cudaStream_t st, const int *kdev) {
    const int lit = literal ? 1 : 0;
    if (first) {
        if (early) cn_launch<true, true>(g, w, k, lit, cfg, st, kdev);
        else cn_launch<true, false>(g, w, k, lit, cfg, st, kdev);
    } else {
        if (early) cn_launch<false, true>(g, w, k, lit, cfg, st, kdev);
        else cn_launch<false, false>(g, w, k, lit, cfg, st, kdev);
    }
    return 1;
}

int launch_bit_node(const Graph &g, const StreamState &w, int k, int L, bool early, const StreamLaunch &cfg,
                    cudaStream_t st, const int *kdev) {
    const dim3 grid(cfg.sms * BN_MINB);
    if (early) k_bn<true><<<grid, BN_T, 0, st>>>(g, w, k, L, kdev, cfg.check_every, cfg.compact ? 1 : 0);
    else k_bn<false><<<grid, BN_T, 0, st>>>(g, w, k, L, kdev, cfg.check_every, 0);
    return 1;
}

int launch_compact(const Graph &g, const StreamState &w, int k, const StreamLaunch &cfg, cudaStream_t st,
                   const int *kdev) {
    k_compact_plan<<<1, 1024, 0, st>>>(w, k, kdev);
    k_compact_move<<<cfg.sms * 4, MV_T, 0, st>>>(g, w);
    return 2;
}

int launch_syndrome(const Graph &g, const StreamState &w, int slot, const float *sfin, const StreamLaunch &cfg,
                    cudaStream_t st) {
    k_syndrome<<<cfg.sms * 4, CTA, 0, st>>>(g, w, slot, sfin);
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

int launch_finalize(const Graph &g, const StreamState &w, int L, int final_slot, const float *sfin, float *posterior,
                    uint8_t *bits, cudaStream_t st) {
    k_finalize<<<grid2((g.n + 32 * SI_SUB - 1) / (32 * SI_SUB), w.Tcap), CTA, 0, st>>>(w, g.n, L, final_slot, sfin,
                                                                                       posterior, bits);
    return 1;
}

int launch_frame_stats(const StreamState &w, int64_t frames, int32_t *iters_out, uint8_t *conv_out,
                       unsigned long long *stats, cudaStream_t st) {
    k_frame_stats<<<(unsigned)std::max<int64_t>(1, (frames + CTA - 1) / CTA), CTA, 0, st>>>(w, frames, iters_out,
                                                                                           conv_out, stats);
    return 1;
}

}  // namespace ldpc
