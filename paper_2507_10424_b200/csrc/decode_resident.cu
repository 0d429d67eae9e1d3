// decode_resident.cu -- the SMEM-resident schedule: one persistent CTA per SM decodes S frames at a
// time with the whole per-frame state in shared memory, and refills a frame slot the moment its
// frame stops (per-frame early stop of Alg. 1, without batch-level waste).
//
// Per CTA, frame-interleaved over S slots (a lane owns 4 consecutive slots of one row or column):
//   s    [n][S]  fp32          soft vector (Eq. sCalculation)
//   min0 [m][S]  fp32          Observation 1's minimum; SIGN BIT = the row's sign parity
//                              (Obs. 2) x (-1)^{d_i} (reading A1)
//   min1 [m][S]  fp32          Observation 1's second minimum, same sign bit
//   eb   [m][LR][DMP] u8       edge bytes: byte (i, l, p) = sign nibble (bit v: sign of lambda_e = s_j -
//                              eta_e for edge p of row i and slot 4l + v) | isloc nibble << 4 (bit v: p is
//                              min0Location of slot 4l + v); the lane that owns slots 4l..4l+3 of row i
//                              owns its DMP = ceil(dmax / 8) * 8 bytes (read and written 8 at a time)
// eta_e = (isloc ? min1 : min0) with its sign bit XORed with the stored bit: one FSEL and one LOP3 per
// slot-edge, the select predicates of 4 slots from one byte (the layout of the streaming schedule's edge
// blocks; it replaced round 1's location bytes and row-transposed sign words: C2 9.80 -> 10.77 Gbps).
// Zeros of s are kept as -0.0 (same slice and sign() under reading A12), so the decision of a slot is
// the complement of the IEEE sign bit of s and the syndrome is a XOR of sign bits.
// plus the Tanner graph itself as 16-bit lists (N_i, M_j).  r lives in a global scratch
// [CTA][n][S] (L2-resident) read once per column per body.  Loop per round:
//   A  finish stopped slots (k, isCodeword, counters) and refill empty slots from a global counter
//   B  stage new frames into their slots (s = r; eta^prev = 0 is applied by the next check-node pass)
//   C  check-node pass over all rows + syndrome of b = slice(s) of every slot
//   D  per slot: stop (codeword, or k = L) -> write b and s; else bit-node pass s = sum eta + r
// Every sweep uses the same lane mapping (4 slots of one row/column per lane, 16-byte accesses), so
// no sweep has shared-memory bank conflicts beyond the row/column gather itself.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "ldpc_internal.cuh"

namespace ldpc {

namespace {

constexpr unsigned FULLM = 0xffffffffu;


struct Layout {
    size_t s, m0, m1, eb, rp, cp, col, rec, rec2, meta, total;
};

constexpr size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }

constexpr int META_INTS = 8 * 32 + 16;

// Edge bytes per lane and row: DMP = ceil(dm / 8) * 8 bytes (8-byte chunks), see eb_dmp.
// compact: the bit node's per-edge records are a u16 row offset and a u8 position (3 B per edge instead
// of 8: the edge-byte index is recomputed from them), for codes that fit no other way (C5 size)
__host__ __device__ constexpr int eb_dmp(int dm) { return (dm + 7) / 8 * 8; }

Layout layout_for(int S, int m, int n, int E, int dm, bool compact = false, bool gg = false) {
    Layout L{};
    if (gg) E = 0;  // global-graph mode: the edge lists stay in global memory (L2)
    size_t o = 0;
    L.s = o;    o = a16(o + (size_t)n * S * 4);
    L.m0 = o;   o = a16(o + (size_t)m * S * 4);
    L.m1 = o;   o = a16(o + (size_t)m * S * 4);
    L.eb = o;   o = a16(o + (size_t)m * (S / 4) * eb_dmp(dm));
    L.rp = o;   o = a16(o + (size_t)(m + 1) * 2);
    L.cp = o;   o = a16(o + (size_t)(n + 1) * 2);
    L.col = o;  o = a16(o + (size_t)E * 2);
    L.rec = o;  o = a16(o + (size_t)E * (compact ? 2 : 8));  // compact: u16 row offset; else uint2 {state, byte}
    L.rec2 = o; o = a16(o + (size_t)E * (compact ? 1 : 0));  // compact: u8 position
    L.meta = o; o = a16(o + (size_t)META_INTS * 4 + 8 * 8);
    L.total = o;
    return L;
}

struct ResArgs {
    Graph g;
    const float *llr;
    int64_t frames;
    int L, T, early, literal, dm;
    int dc, dv;  // > 0: every row has degree dc and every column degree dv (regular code)
    int compact;  // bit-node records in the compact form (see layout_for)
    int gg;       // Tanner-graph edge lists read from global memory
    int any_degree;  // force the any-degree check-node instance (tests)
    float *post;
    uint8_t *bits;
    int32_t *iters;
    uint8_t *conv;
    unsigned long long *stats;
    int *counter;
    float *rs;
    Layout lay;
};

__device__ __forceinline__ float f4c(const float4 &a, int v) { return v == 0 ? a.x : v == 1 ? a.y : v == 2 ? a.z : a.w; }
__device__ __forceinline__ void f4s(float4 &a, int v, float x) {
    if (v == 0) a.x = x;
    else if (v == 1) a.y = x;
    else if (v == 2) a.z = x;
    else a.w = x;
}

// Check-node update of G rows (one per row group of the warp) for the 4 slots of this lane.
// HAS: rows of the warp may have different degrees (irregular H), lanes past their degree idle.
// fm: this lane's fresh slots (eta^prev = 0: their stored min0 = min1 = +0, so eta^prev = +-0 and
// lambda = s - (+-0) has the magnitude and sign() of s, s being -0 rather than +0 for zero).
// sgw: this lane's sign words of row i (sgw[q * LR] = edges 8q..8q+7): read as eta^prev's signs and
// overwritten with the new ones (each lane owns its words: no ballot, no synchronisation).
#ifndef RES_ANY_UNROLL
#define RES_ANY_UNROLL 1  // edge pairs per unrolled step of the any-degree check-node pass (4: 1 % slower)
#endif
constexpr int kAnyUnroll = RES_ANY_UNROLL;  // (#pragma unroll does not expand macros)
#ifndef RES_TREE
#define RES_TREE 1  // rows of <= 8 edges: pair tournament after all lambdas, isloc = (|lambda| == min0)
#endif

// min(a, b, c) in one FMNMX3 (sm_100)
__device__ __forceinline__ float fmin3f(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

__device__ __forceinline__ float flip31(float mag, uint32_t bit31) {
    return __uint_as_float(__float_as_uint(mag) ^ (bit31 & 0x80000000u));
}

// The 8 edge bytes of a chunk from its sign word sw (bit 4u+v: sign of lambda, edge u, slot v) and isloc
// word lm (same layout): byte u = sign nibble | isloc nibble << 4, one 8-byte store (all 8 bytes of the
// chunk; bytes past the row's degree are never read).
__device__ __forceinline__ void res_store_chunk(uint8_t *p, uint32_t sw, uint32_t lm) {
    const uint32_t ze = (sw & 0x0f0f0f0fu) | ((lm & 0x0f0f0f0fu) << 4);  // edges 0, 2, 4, 6
    const uint32_t zo = ((sw >> 4) & 0x0f0f0f0fu) | (lm & 0xf0f0f0f0u);  // edges 1, 3, 5, 7
    *reinterpret_cast<uint2 *>(p) = make_uint2(__byte_perm(ze, zo, 0x5140), __byte_perm(ze, zo, 0x7362));
}

__device__ __forceinline__ int colat(const uint16_t *c, int e) { return c[e]; }
__device__ __forceinline__ int colat(const int *c, int e) { return __ldg(c + e); }

template <int S, bool HAS, int DC, typename CT>
__device__ __forceinline__ void cn_rows(const float *__restrict__ s, float *mn0, float *mn1, uint8_t *__restrict__ ebr,
                                        const CT *col, int i, bool valid, int ra, int d, int dmax, int l,
                                        unsigned fm, bool corr, unsigned &syn_acc) {
    const float INF = __int_as_float(0x7f800000);
    const int q0 = 4 * l;
    float4 om0 = make_float4(0.f, 0.f, 0.f, 0.f), om1 = om0;
    const int ca = i * S + q0;
    if (valid) {
        om0 = *reinterpret_cast<const float4 *>(mn0 + ca);
        om1 = *reinterpret_cast<const float4 *>(mn1 + ca);
        if (fm) {  // fresh slots start from eta = 0: min0 = min1 = +0 (eta^prev = +-0 whatever the edge byte)
            if (fm & 1u) { om0.x = 0.f; om1.x = 0.f; }
            if (fm & 2u) { om0.y = 0.f; om1.y = 0.f; }
            if (fm & 4u) { om0.z = 0.f; om1.z = 0.f; }
            if (fm & 8u) { om0.w = 0.f; om1.w = 0.f; }
        }
    }
    float nm0[4] = {INF, INF, INF, INF}, nm1[4] = {INF, INF, INF, INF};
    int nloc[4] = {0, 0, 0, 0};
    uint32_t synw[4] = {0u, 0u, 0u, 0u};  // XOR of the sign bits of s over the row: bit 31 = XOR of (1 - b_j)
    // the lane's edge bytes of the row (sign nibble | isloc nibble << 4), 8 per chunk (one 8-byte access);
    // new sign bits are pushed into wn by one funnel shift per slot-edge, in (p, v) order, and a chunk's
    // word is bit-reversed into bit 4(p%8)+v
    uint2 ob = make_uint2(0u, 0u);
    uint32_t wn = 0u, pf = 0u;
    // DC > 0: the warp's rows have at most DC edges, DC of them without HAS (unrolled); DC == 0: any degree
    const int pe = DC > 0 ? DC : dmax;
    // Edges in pairs (p, p+1; p even, so a pair never straddles a chunk): the pair's smaller and larger
    // |lambda| (sm, tm) update the row state with nm0' = min(nm0, sm), nm1' = min3(nm1, max(nm0, sm), tm)
    // (FMNMX3) and loc' = sm < nm0 ? (b < a ? p+1 : p) : loc -- the same first strict minimum (A13) and
    // second minimum as the edge-by-edge update in fewer ALU operations; the decision parity takes both
    // edges in one 3-input XOR.  An absent edge enters as |lambda| = +inf, sign bit 0, parity 0.
#if RES_TREE
    if constexpr (DC > 0 && DC <= 8) {
        // One chunk (rows of at most 8 edges): every lambda of the row first, then min0 / min1 by a pair
        // tournament and the min0Location bits as the edges whose |lambda| equals min0 (every edge of a
        // tie: under a tie min1 = min0, same value and sign bit, so eta_e is the same; reading A13) -- the
        // check node of the streaming schedule (decode_stream.cu, cn_compute) in the resident layout.
        if (valid) ob = *reinterpret_cast<const uint2 *>(ebr);
        float ax[DC][4];
        uint32_t iw = 0u;
#pragma unroll
        for (int p = 0; p < DC; p++) {
            const bool hp = HAS ? (p < d) : true;
            const int j = hp ? colat(col, ra + p) : 0;
            const float4 sv = *reinterpret_cast<const float4 *>(s + j * S + q0);
            const uint32_t b = ((p & 4) ? ob.y : ob.x) >> (8 * (p & 3));
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const float sj = f4c(sv, v);
                const float mg = (b & (16u << v)) ? f4c(om1, v) : f4c(om0, v);  // Obs. 1 (+ row parity)
                const float x = __fadd_rn(__fsub_rn(sj, flip31(mg, b << (31 - v))), 0.0f);  // lambda, zero -> +0
                ax[p][v] = hp ? fabsf(x) : INF;
                wn = __funnelshift_l(hp ? __float_as_uint(x) : 0u, wn, 1);
                synw[v] ^= hp ? __float_as_uint(sj) : 0u;  // slice(s_j) = 0 iff sign bit
            }
        }
#pragma unroll
        for (int v = 0; v < 4; v++) {
            float lo = fminf(ax[0][v], ax[1][v]), hi = fmaxf(ax[0][v], ax[1][v]);
#pragma unroll
            for (int p = 2; p + 1 < DC; p += 2) {
                const float l2 = fminf(ax[p][v], ax[p + 1][v]), h2 = fmaxf(ax[p][v], ax[p + 1][v]);
                hi = fmin3f(hi, h2, fmaxf(lo, l2));
                lo = fminf(lo, l2);
            }
            if (DC & 1) {
                hi = fminf(hi, fmaxf(lo, ax[DC - 1][v]));
                lo = fminf(lo, ax[DC - 1][v]);
            }
            nm0[v] = lo;
            nm1[v] = hi;
        }
#pragma unroll
        for (int p = 0; p < DC; p++)
#pragma unroll
            for (int v = 0; v < 4; v++) iw = __funnelshift_l(__float_as_uint(__fsub_rn(nm0[v], ax[p][v])), iw, 1);
        wn = DC == 8 ? __brev(wn) : __brev(wn) >> (32 - 4 * DC);
        pf = wn;
        const uint32_t lm = DC == 8 ? __brev(~iw) : __brev(~iw) >> (32 - 4 * DC);  // bit 4p+v: isloc
        if (valid) res_store_chunk(ebr, wn, lm);
    } else
#endif
    {
#pragma unroll(DC > 0 ? (DC + 1) / 2 : kAnyUnroll)
        for (int p = 0; p < pe; p += 2) {
            if ((p & 7) == 0) {
                if (p > 0) {  // the finished chunk: its bytes with the sign nibbles (isloc merged at the row end)
                    wn = __brev(wn);
                    pf ^= wn;
                    if (valid) res_store_chunk(ebr + p - 8, wn, 0u);
                    wn = 0u;
                }
                if (valid) ob = *reinterpret_cast<const uint2 *>(ebr + p);
            }
            const bool inb = p + 1 < pe;
            const bool ha = HAS ? (p < d) : true, hb = inb && (HAS ? (p + 1 < d) : true);
            const int ja = ha ? colat(col, ra + p) : 0, jb = hb ? colat(col, ra + p + 1) : 0;
            const float4 sva = *reinterpret_cast<const float4 *>(s + ja * S + q0);
            const float4 svb = *reinterpret_cast<const float4 *>(s + jb * S + q0);
            const uint32_t ow = (p & 4) ? ob.y : ob.x;
            const uint32_t ba = ow >> (8 * (p & 3)), bb = ow >> (8 * ((p + 1) & 3));
            float xa[4], xb[4];
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const float sa = f4c(sva, v), sb = f4c(svb, v);
                const float ma = (ba & (16u << v)) ? f4c(om1, v) : f4c(om0, v);  // Obs. 1 (+ row parity)
                const float mb = (bb & (16u << v)) ? f4c(om1, v) : f4c(om0, v);
                // lambda - eta^prev; + 0 makes a zero lambda +0 (s may be -0), so its IEEE sign bit is
                // sign(0) = +1; the add runs on the otherwise idle FMA pipe
                xa[v] = __fadd_rn(__fsub_rn(sa, flip31(ma, ba << (31 - v))), 0.0f);
                xb[v] = __fadd_rn(__fsub_rn(sb, flip31(mb, bb << (31 - v))), 0.0f);
                synw[v] ^= (ha ? __float_as_uint(sa) : 0u) ^ (hb ? __float_as_uint(sb) : 0u);  // slice(s_j) = 0 iff sign bit
            }
#pragma unroll
            for (int v = 0; v < 4; v++) wn = __funnelshift_l(ha ? __float_as_uint(xa[v]) : 0u, wn, 1);
            if (inb) {
#pragma unroll
                for (int v = 0; v < 4; v++) wn = __funnelshift_l(hb ? __float_as_uint(xb[v]) : 0u, wn, 1);
            }
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const float a = ha ? fabsf(xa[v]) : INF, b = hb ? fabsf(xb[v]) : INF;
                const float sm = fminf(a, b), tm = fmaxf(a, b);
                const int lp = b < a ? p + 1 : p;
                const bool lt = sm < nm0[v];
                nm1[v] = fmin3f(nm1[v], fmaxf(nm0[v], sm), tm);
                nm0[v] = fminf(nm0[v], sm);
                nloc[v] = lt ? lp : nloc[v];
            }
        }
        {
            const int last = (pe - 1) & ~7;            // first edge of the last chunk
            const int pushed = 4 * (pe - last);        // slot-edges in the last chunk
            wn = pushed == 32 ? __brev(wn) : __brev(wn) >> (32 - pushed);
            pf ^= wn;
            if (valid) {
                if ((DC > 0 && DC <= 8) || pe <= 8) {  // one chunk (regular codes of degree <= 8): isloc merged before the only store
                    const uint32_t lm = (1u << (4 * nloc[0])) | (2u << (4 * nloc[1])) | (4u << (4 * nloc[2])) |
                                        (8u << (4 * nloc[3]));
                    res_store_chunk(ebr, wn, lm);
                } else {
                    res_store_chunk(ebr + last, wn, 0u);
#pragma unroll
                    for (int v = 0; v < 4; v++) ebr[nloc[v]] |= (uint8_t)(16u << v);  // this thread wrote them
                }
            }
        }
    }
    if (valid) {
        // this lane's row sign parity per slot (XOR of bits v, v+4, ... of the sign words), times
        // (-1)^{d_i} under the CORRECTED rule (reading A1)
        uint32_t pw = pf ^ (pf >> 16);
        pw ^= pw >> 8;
        pw ^= pw >> 4;
        pw ^= (corr && (d & 1)) ? 0xfu : 0u;
        const uint32_t sb[4] = {pw << 31, (pw << 30) & 0x80000000u, (pw << 29) & 0x80000000u,
                                (pw << 28) & 0x80000000u};
        *reinterpret_cast<float4 *>(mn0 + ca) =
            make_float4(__uint_as_float(__float_as_uint(nm0[0]) | sb[0]), __uint_as_float(__float_as_uint(nm0[1]) | sb[1]),
                        __uint_as_float(__float_as_uint(nm0[2]) | sb[2]), __uint_as_float(__float_as_uint(nm0[3]) | sb[3]));
        *reinterpret_cast<float4 *>(mn1 + ca) =
            make_float4(__uint_as_float(__float_as_uint(nm1[0]) | sb[0]), __uint_as_float(__float_as_uint(nm1[1]) | sb[1]),
                        __uint_as_float(__float_as_uint(nm1[2]) | sb[2]), __uint_as_float(__float_as_uint(nm1[3]) | sb[3]));
        // row unsatisfied iff XOR_j b_j = 1, with XOR_j b_j = d_i mod 2 xor XOR_j (1 - b_j)
        const uint32_t dp = (uint32_t)(d & 1);
        syn_acc |= (((synw[0] >> 31) ^ dp) | (((synw[1] >> 31) ^ dp) << 1) | (((synw[2] >> 31) ^ dp) << 2) |
                    (((synw[3] >> 31) ^ dp) << 3));
    }
}

// Lane layout: a lane owns 4 consecutive slots (float4) of one row or column; LR = S/4 lanes cover a
// row, G = 32/LR rows per warp.  Bit of slot q = 4*l + v inside an S-bit sign word: v*LR + l.
template <int S, int RT, int DC, int DV, bool CMP, bool GG = false>
__global__ void __launch_bounds__(RT, RT == 128 ? 4 : RT == 256 ? (S == 4 ? 3 : 2) : RT == 384 ? 2 : 1) k_resident(ResArgs a) {
    constexpr int NWARP = RT / 32;
    constexpr int LR = S / 4;
    constexpr int G = 32 / LR;
    extern __shared__ __align__(16) unsigned char sm[];
    const int m = a.g.m, n = a.g.n, E = a.g.E;
    float *s = reinterpret_cast<float *>(sm + a.lay.s);
    float *mn0 = reinterpret_cast<float *>(sm + a.lay.m0);
    float *mn1 = reinterpret_cast<float *>(sm + a.lay.m1);
    uint8_t *ebt = sm + a.lay.eb;
    const int DMP = eb_dmp(a.dm);  // edge bytes per lane and row
    uint16_t *rp = reinterpret_cast<uint16_t *>(sm + a.lay.rp);
    uint16_t *cp = reinterpret_cast<uint16_t *>(sm + a.lay.cp);
    uint16_t *col = reinterpret_cast<uint16_t *>(sm + a.lay.col);
    // the check-node pass's column lists: shared memory, or (GG) the ingested int32 lists in global memory
    const typename std::conditional<GG, int, uint16_t>::type *colp;
    if constexpr (GG) colp = a.g.col_idx;
    else colp = col;
    uint32_t *rec = reinterpret_cast<uint32_t *>(sm + a.lay.rec);
    uint32_t *rec2 = reinterpret_cast<uint32_t *>(sm + a.lay.rec2);
    int *meta = reinterpret_cast<int *>(sm + a.lay.meta);
    int *slot_f = meta;            // frame index of the slot, -1 = empty
    int *slot_k = meta + 32;       // completed loop bodies
    int *slot_be = meta + 64;      // ones of b (bit errors vs the all-zero codeword)
    int *slot_raw = meta + 96;     // r_j > 0 count
    int *slot_nz = meta + 128;     // some |s_j| <= 1e-4 (frame that stopped in the last pass)
    int *slot_fout = meta + 160;   // frame index of the slot's stopping frame (outputs of this pass)
    int *slot_pend = meta + 192;   // 1 + isCodeword of a stopped frame whose error counts are pending
    // ctl: [0] unsat, [1] fresh, [2] active (continuing | fresh), [3] exhausted, [4] stopping, [5] continuing
    unsigned *ctl = reinterpret_cast<unsigned *>(meta + 256);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sub = lane / LR, l = lane % LR;  // row group inside the warp, lane inside the row
    const int q0 = 4 * l;                      // first slot of this lane
    float *rs = a.rs + (size_t)blockIdx.x * n * S;
    const bool corr = !a.literal;

    // ---- the Tanner graph into shared memory (16-bit lists)
    for (int q = tid; q <= m; q += RT) rp[q] = (uint16_t)__ldg(a.g.row_ptr + q);
    for (int q = tid; q <= n; q += RT) cp[q] = (uint16_t)__ldg(a.g.col_ptr + q);
    for (int e = tid; e < (GG ? 0 : E); e += RT) {
        col[e] = (uint16_t)__ldg(a.g.col_idx + e);
        const int4 be = __ldg(a.g.bn_edge + e);  // {edge id, row, pos, parity}
        if (CMP) {  // u16 row offset, u8 position
            reinterpret_cast<uint16_t *>(rec)[e] = (uint16_t)(be.y * S);
            reinterpret_cast<uint8_t *>(rec2)[e] = (uint8_t)be.z;
            continue;
        }
        // {first state element of row i (the lane adds its slot offset), the edge's byte for lane 0 (the
        // lane adds l * DMP)}: one 8-byte shared load per edge in the bit-node pass
        reinterpret_cast<uint2 *>(rec)[e] = make_uint2((uint32_t)be.y * S, (uint32_t)(be.y * LR * DMP + be.z));
    }
    if (tid < 32) {
        slot_f[tid] = -1;
        slot_k[tid] = 0;
        slot_be[tid] = 0;
        slot_raw[tid] = 0;
        slot_nz[tid] = 0;
        slot_fout[tid] = -1;
        slot_pend[tid] = 0;
    }
    if (tid < 8) ctl[tid] = 0;
    unsigned long long acc_stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // warp 0, lane = slot
    __syncthreads();

    // Per pass: C (check node + syndrome), then A (warp 0: stop / continue / refill the slots), then one
    // column sweep D that writes the outputs of the stopping frames, runs the bit node of the continuing
    // ones and stages the new frames (s = r) -- so a refill costs no extra sweep and no extra barrier.
    // The first A and D (before the first C) only stage the first frames.
    unsigned active = 0;
    for (int pass = 0;; pass++) {
        if (pass > 0) {
            const unsigned fresh_prev = ctl[1];
            const unsigned fm = (fresh_prev >> q0) & 0xfu;  // this lane's fresh slots (eta^prev = 0)
            // ---------------- C: check-node pass + syndrome of b = slice(s)
            unsigned syn_acc = 0;  // bit v: slot q0+v has an unsatisfied check
            for (int rb = warp * G; rb < m; rb += NWARP * G) {
                const int i = rb + sub;
                const bool valid = i < m;
                const int ra = DC > 0 ? i * DC : (valid ? rp[i] : 0);
                const int d = DC > 0 ? (valid ? DC : 0) : (valid ? (int)rp[i + 1] - ra : 0);
                const int dmax = DC > 0 ? DC : __reduce_max_sync(FULLM, d);
                uint8_t *ebr = ebt + ((size_t)(valid ? i : 0) * LR + l) * DMP;
#define CN_ROWS_(H, K) cn_rows<S, H, K>(s, mn0, mn1, ebr, colp, i, valid, ra, d, dmax, l, fm, corr, syn_acc)
                if (DC > 0 && rb + G <= m) {
                    CN_ROWS_(false, (DC > 0 ? DC : 1));
                } else if (DC < 0) {
                    // rows of degree <= 8, any code: an instance per largest degree of the warp's rows (a
                    // run-time value), unrolled, with per-edge guards only where the warp's degrees differ
                    const bool eq = __all_sync(FULLM, d == dmax);
                    switch (dmax) {
                        case 2: if (eq) CN_ROWS_(false, 2); else CN_ROWS_(true, 2); break;
                        case 3: if (eq) CN_ROWS_(false, 3); else CN_ROWS_(true, 3); break;
                        case 4: if (eq) CN_ROWS_(false, 4); else CN_ROWS_(true, 4); break;
                        case 5: if (eq) CN_ROWS_(false, 5); else CN_ROWS_(true, 5); break;
                        case 6: if (eq) CN_ROWS_(false, 6); else CN_ROWS_(true, 6); break;
                        case 7: if (eq) CN_ROWS_(false, 7); else CN_ROWS_(true, 7); break;
                        case 8: if (eq) CN_ROWS_(false, 8); else CN_ROWS_(true, 8); break;
                        default: CN_ROWS_(true, 0); break;
                    }
                } else if (__all_sync(FULLM, d == dmax)) {
                    CN_ROWS_(false, 0);
                } else {
                    CN_ROWS_(true, 0);
                }
#undef CN_ROWS_
            }
            const unsigned mine = (syn_acc << q0) & active;
            const unsigned wmask = __reduce_or_sync(FULLM, mine);
            if (lane == 0 && wmask) atomicOr(&ctl[0], wmask);
            __syncthreads();
        }
        // ---------------- A: stop / continue / refill (warp 0)
        if (warp == 0) {
            const unsigned uns_all = ctl[0];
            const bool own = lane < S;
            // error counts of the frames that stopped in the previous pass (written by that pass's D)
            if (own && slot_pend[lane]) {
                const int be = slot_be[lane], conv = slot_pend[lane] - 1;
                acc_stats[1] += (unsigned long long)be;
                acc_stats[2] += be > 0;
                acc_stats[3] += (be > 0) && conv;
                acc_stats[6] += slot_nz[lane] != 0;
                slot_be[lane] = 0;
                slot_nz[lane] = 0;
                slot_pend[lane] = 0;
            }
            int f = own ? slot_f[lane] : 0;
            bool fin = false, cont = false;
            if (own && f >= 0 && pass > 0) {
                const int k = slot_k[lane];
                const bool uns = (uns_all >> lane) & 1u;
                // a clean syndrome stops the frame only at a check point k % T == 0
                fin = a.early ? ((!uns && k % a.T == 0) || k == a.L) : (k == a.L);
                if (fin) {
                    const int conv = !uns;
                    if (a.iters) a.iters[f] = k;
                    if (a.conv) a.conv[f] = (uint8_t)conv;
                    acc_stats[0] += 1;
                    acc_stats[4] += (unsigned long long)k;
                    acc_stats[5] += conv;
                    acc_stats[7] += (unsigned long long)slot_raw[lane];
                    slot_fout[lane] = f;
                    slot_pend[lane] = 1 + conv;
                    f = -1;
                } else {
                    slot_k[lane] = k + 1;  // D runs body k + 1
                    cont = true;
                }
            }
            // refill: the free slots take consecutive frames from the global counter
            const bool exhausted = ctl[3] != 0;
            const unsigned freem = __ballot_sync(FULLM, own && f < 0);
            long long base = 0;
            if (lane == 0 && freem && !exhausted) base = atomicAdd(a.counter, __popc(freem));
            base = __shfl_sync(FULLM, base, 0);
            bool take = false;
            if (freem && !exhausted) {
                const long long mine_f = base + __popc(freem & ((1u << lane) - 1u));
                take = own && f < 0 && mine_f < a.frames;
                if (take) {
                    f = (int)mine_f;
                    slot_k[lane] = 0;
                    slot_raw[lane] = 0;
                }
            }
            if (own) slot_f[lane] = f;
            const unsigned fresh = __ballot_sync(FULLM, take), fin_m = __ballot_sync(FULLM, fin),
                           cont_m = __ballot_sync(FULLM, cont);
            __syncwarp();  // every lane has read ctl[] before lane 0 rewrites it
            if (lane == 0) {
                if (freem && !exhausted && base + __popc(freem) >= a.frames) ctl[3] = 1;
                ctl[0] = 0;
                ctl[1] = fresh;
                ctl[2] = fresh | cont_m;
                ctl[4] = fin_m;
                ctl[5] = cont_m;
            }
        }
        __syncthreads();
        active = ctl[2];
        const unsigned fin_mask = ctl[4], cont_mask = ctl[5], fresh_mask = ctl[1];
        // ---------------- D: outputs of the stopping frames, bit node of the continuing ones, staging of
        //                     the new ones (s = r), in one column sweep
        if (fin_mask | active) {
            const unsigned cm = (cont_mask >> q0) & 0xfu;   // continuing slots of this lane
            const unsigned fk = (fin_mask >> q0) & 0xfu;    // stopping slots of this lane
            const unsigned fw = (fresh_mask >> q0) & 0xfu;  // new frames of this lane
            int64_t fo[4], fr[4];
#pragma unroll
            for (int v = 0; v < 4; v++) {
                fo[v] = (int64_t)slot_fout[q0 + v] * n;
                fr[v] = (int64_t)slot_f[q0 + v] * n;
            }
            int be[4] = {0, 0, 0, 0}, raw[4] = {0, 0, 0, 0};
            unsigned nz = 0;
            for (int cb = warp * G; cb < n; cb += NWARP * G) {
                const int j = cb + sub;
                if (j >= n || !(cm | fk | fw)) continue;
                float *sp = s + j * S + q0;
                // global loads first (r of the continuing slots, the channel values of the new frames), so
                // their latency overlaps the outputs and the bit-node pass below (ncu: the staging and the
                // final add were waiting on them)
                float4 rj = make_float4(0.f, 0.f, 0.f, 0.f);
                if (cm) rj = *reinterpret_cast<const float4 *>(rs + (size_t)j * S + q0);
                float xs[4] = {0.f, 0.f, 0.f, 0.f};
                if (fw) {
#pragma unroll
                    for (int v = 0; v < 4; v++)
                        if ((fw >> v) & 1u) xs[v] = __ldg(a.llr + fr[v] + j);
                }
                // the old s is needed unless all four slots continue (their s is overwritten)
                float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                if (cm != 0xfu) o = *reinterpret_cast<const float4 *>(sp);
                if (fk) {
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        if ((fk >> v) & 1u) {
                            const float x = f4c(o, v);
                            const bool b = x > 0.f;  // Eq. slice
                            if (a.post) a.post[fo[v] + j] = x;
                            if (a.bits) a.bits[fo[v] + j] = (uint8_t)b;
                            be[v] += b;
                            nz |= (unsigned)(fabsf(x) <= 1e-4f) << v;
                        }
                    }
                }
                if (cm) {
                    const int c0 = DV > 0 ? j * DV : cp[j], dv = DV > 0 ? DV : (int)cp[j + 1] - c0;
                    float acc[4] = {0.f, 0.f, 0.f, 0.f};
                    for (int q3 = 0; q3 < dv; q3 += 3) {  // chunks of 3 edges: no remainder loop for d_v = 3
#pragma unroll
                        for (int u = 0; u < 3; u++) {
                            if (q3 + u < dv) {
                                int ca, bi;  // state index of row i for this lane, index of its edge byte
                                if (GG) {  // {e, i, p, -} from global memory (L2)
                                    const int4 be = __ldg(a.g.bn_edge + c0 + q3 + u);
                                    ca = be.y * S + q0;
                                    bi = (be.y * LR + l) * DMP + be.z;
                                } else if (CMP) {
                                    const int ro = reinterpret_cast<const uint16_t *>(rec)[c0 + q3 + u];
                                    const int pq = reinterpret_cast<const uint8_t *>(rec2)[c0 + q3 + u];
                                    ca = ro + q0;
                                    bi = (ro / S * LR + l) * DMP + pq;
                                } else {
                                    const uint2 r12 = reinterpret_cast<const uint2 *>(rec)[c0 + q3 + u];
                                    ca = (int)r12.x + q0;
                                    bi = (int)r12.y + l * DMP;
                                }
                                const float4 m0 = *reinterpret_cast<const float4 *>(mn0 + ca);
                                const float4 m1 = *reinterpret_cast<const float4 *>(mn1 + ca);
                                const uint32_t b = ebt[bi];  // sign nibble | isloc nibble << 4
#pragma unroll
                                for (int v = 0; v < 4; v++) {  // ascending rows from +0.0 (A14)
                                    const float mg = (b & (16u << v)) ? f4c(m1, v) : f4c(m0, v);  // Obs. 1
                                    acc[v] = acc[v] + flip31(mg, b << (31 - v));
                                }
                            }
                        }
                    }
                    const float n0 = acc[0] + rj.x, n1 = acc[1] + rj.y, n2 = acc[2] + rj.z, n3 = acc[3] + rj.w;
                    if (cm & 1u) o.x = n0 == 0.f ? -0.f : n0;  // zeros of s are kept as -0 (A12)
                    if (cm & 2u) o.y = n1 == 0.f ? -0.f : n1;
                    if (cm & 4u) o.z = n2 == 0.f ? -0.f : n2;
                    if (cm & 8u) o.w = n3 == 0.f ? -0.f : n3;
                }
                if (fw) {
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        if ((fw >> v) & 1u) {
                            const float x = xs[v];
                            f4s(o, v, x == 0.f ? -0.f : x);  // zeros of s are kept as -0 (A12)
                            rs[(size_t)j * S + q0 + v] = x;
                            raw[v] += x > 0.f;
                        }
                    }
                }
                if (cm | fw) *reinterpret_cast<float4 *>(sp) = o;
            }
            // per-slot counts: reduce over the row groups of the warp, then one atomic per slot (the
            // condition is CTA-uniform: every lane of the warp takes part in the shuffles)
            if (fin_mask | fresh_mask) {
#pragma unroll
                for (int v = 0; v < 4; v++) {
                    int x = be[v], y = raw[v];
                    for (int o = LR; o < 32; o <<= 1) {
                        x += __shfl_xor_sync(FULLM, x, o);
                        y += __shfl_xor_sync(FULLM, y, o);
                    }
                    if (sub == 0 && x) atomicAdd(&slot_be[q0 + v], x);
                    if (sub == 0 && y) atomicAdd(&slot_raw[q0 + v], y);
                }
                unsigned z = nz;
                for (int o = LR; o < 32; o <<= 1) z |= __shfl_xor_sync(FULLM, z, o);
                if (sub == 0 && z)
#pragma unroll
                    for (int v = 0; v < 4; v++)
                        if ((z >> v) & 1u) slot_nz[q0 + v] = 1;
            }
        }
        __syncthreads();
        if (!active) break;
    }
    // error counts of the frames that stopped in the last pass
    if (warp == 0 && lane < S && slot_pend[lane]) {
        const int be = slot_be[lane], conv = slot_pend[lane] - 1;
        acc_stats[1] += (unsigned long long)be;
        acc_stats[2] += be > 0;
        acc_stats[3] += (be > 0) && conv;
        acc_stats[6] += slot_nz[lane] != 0;
    }

    // ---- counters: warp 0 holds them per slot
    if (warp == 0 && a.stats) {
#pragma unroll
        for (int q = 0; q < 8; q++) {
            unsigned long long x = acc_stats[q];
            for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULLM, x, o);
            if (lane == 0 && x) atomicAdd(a.stats + q, x);
        }
    }
}

int max_smem_optin(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    return v;
}

template <int S, int RT, bool CMP>
void launch_c(const ResArgs &args, int ctas, size_t smem, cudaStream_t st) {
    // regular (3,6) codes (C1, C2, C5): degree-specialised kernel (fully unrolled row and column loops)
    if (args.dc == 6 && args.dv == 3) {
        cudaFuncSetAttribute(k_resident<S, RT, 6, 3, CMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_resident<S, RT, 6, 3, CMP><<<ctas, RT, smem, st>>>(args);
        return;
    }
    // rows of degree <= 8 (most codes): the check-node pass unrolled over at most 4 edge pairs
    if (args.dm <= 8 && !args.any_degree) {
        cudaFuncSetAttribute(k_resident<S, RT, -8, 0, CMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_resident<S, RT, -8, 0, CMP><<<ctas, RT, smem, st>>>(args);
        return;
    }
    cudaFuncSetAttribute(k_resident<S, RT, 0, 0, CMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_resident<S, RT, 0, 0, CMP><<<ctas, RT, smem, st>>>(args);
}

// global-graph mode (codes whose per-slot state fills shared memory, C6 size): S <= 8, 512 threads
template <int S>
void launch_gg(const ResArgs &args, int ctas, size_t smem, cudaStream_t st) {
    if (args.dm <= 8 && !args.any_degree) {
        cudaFuncSetAttribute(k_resident<S, 512, -8, 0, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_resident<S, 512, -8, 0, false, true><<<ctas, 512, smem, st>>>(args);
        return;
    }
    cudaFuncSetAttribute(k_resident<S, 512, 0, 0, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_resident<S, 512, 0, 0, false, true><<<ctas, 512, smem, st>>>(args);
}

template <int S, int RT>
void launch_s(const ResArgs &args, int ctas, size_t smem, cudaStream_t st) {
    if (args.gg) {  // the planner only picks the global-graph mode with S <= 8 and 512 threads
        if constexpr (S <= 8 && RT == 512) launch_gg<S>(args, ctas, smem, st);
        return;
    }
    if (args.compact) {  // the planner only picks compact records with S <= 8 and 256 / 512 threads
        if constexpr (S <= 8 && (RT == 256 || RT == 512)) launch_c<S, RT, true>(args, ctas, smem, st);
        return;
    }
    launch_c<S, RT, false>(args, ctas, smem, st);
}

template <int S>
void launch_t(const ResArgs &args, int threads, int ctas, size_t smem, cudaStream_t st) {
    if (threads == 1024) launch_s<S, 1024>(args, ctas, smem, st);
    else if (threads == 256) launch_s<S, 256>(args, ctas, smem, st);
    else if (threads == 384) launch_s<S, 384>(args, ctas, smem, st);
    else if (threads == 128) launch_s<S, 128>(args, ctas, smem, st);
    else launch_s<S, 512>(args, ctas, smem, st);
}

}  // namespace

ResidentPlan plan_resident(const HostGraph &g, bool loc16, int device) {
    const int dm = std::max(1, g.max_row_deg);
    (void)loc16;
    ResidentPlan rp;
    if (g.n >= 65535 || g.m >= 65535 || g.E >= 65535 || g.E == 0 || dm > 254) return rp;  // u16 lists, u8 positions
    const int cap = max_smem_optin(device);
    int sms = 0, sm_smem = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    if (cap <= 0 || sms <= 0) return rp;
    int force_s = 0, force_t = 0;
    if (const char *e = getenv("LDPC_RES_SLOTS")) force_s = atoi(e);
    if (const char *e = getenv("LDPC_RES_THREADS")) force_t = atoi(e);
    // Prefer the largest S with two CTAs per SM (their phases interleave: measured 3-12 % faster on
    // the C2 code than one CTA of 2S slots), else the largest S with one CTA per SM.
    // A third pass tries the compact bit-node records (codes of the C5 size: 2048 x 4096 with S = 4).
    // LDPC_RES_COMPACT=1 forces the compact records (tests; they are bit-identical).
    for (int pass = getenv("LDPC_RES_COMPACT") ? 2 : 0; pass < 3 && !rp.ok; pass++) {
        const bool compact = pass == 2;
        if (compact && getenv("LDPC_RES_NO_COMPACT")) break;
        for (int S : {32, 16, 8, 4}) {
            if (force_s && S != force_s) continue;
            if (compact && (S > 8 || (int64_t)g.m * S > 65535)) continue;
            const Layout L = layout_for(S, g.m, g.n, g.E, dm, compact);
            if (L.total > (size_t)cap) continue;
            const int per_sm = std::max(1, std::min(S == 4 ? 3 : 2, sm_smem / (int)(L.total + 1024)));
            if (pass == 0 && per_sm < 2 && !force_s) continue;
            rp.ok = true;
            rp.compact = compact;
            rp.slots = S;
            rp.dm = dm;
            rp.dv = g.max_col_deg;
            rp.regular = (int64_t)g.E == (int64_t)g.m * dm && (int64_t)g.E == (int64_t)g.n * g.max_col_deg;
            rp.smem = L.total;
            rp.threads = per_sm >= 2 ? 256 : 512;
            if (force_t == 128 || force_t == 256 || force_t == 384 || force_t == 512 || force_t == 1024)
                rp.threads = force_t;
            if (compact && rp.threads != 256) rp.threads = 512;  // compact records: 256- or 512-thread kernels only
            const int fit = rp.threads == 128   ? per_sm
                            : rp.threads == 256 ? std::min(per_sm, S == 4 ? 3 : 2)
                            : rp.threads == 384 ? std::min(per_sm, 2)
                                                : 1;
            rp.ctas = sms * fit;
            break;
        }
    }
    // Optional: the per-slot state alone in shared memory, the edge lists read from global memory
    // (L2-resident; C6: 1022 x 8176, d_c = 32, S = 4 in one 512-thread CTA per SM).  Measured slower than
    // the streaming schedule on C6 (1.62 against 2.46 Gbps: 4 frames per SM and L2 latency on every edge
    // list), so only LDPC_RES_GG=1 selects it (tests, A/B); parity-green.
    const char *gge = getenv("LDPC_RES_GG");
    const bool gg_force = gge && atoi(gge) == 1;
    if (gg_force) rp = ResidentPlan{};
    if (!rp.ok && gg_force) {
        for (int S : {8, 4}) {
            if (force_s && S != force_s) continue;
            const Layout L = layout_for(S, g.m, g.n, g.E, dm, false, true);
            if (L.total > (size_t)cap) continue;
            rp.ok = true;
            rp.global_graph = true;
            rp.slots = S;
            rp.dm = dm;
            rp.dv = g.max_col_deg;
            rp.regular = false;
            rp.smem = L.total;
            rp.threads = 512;
            rp.ctas = sms;
            break;
        }
    }
    return rp;
}

// rs scratch is carved after the two counter ints of work_counter's allocation owner (runtime.cu)
int launch_resident(const Graph &g, const ResidentPlan &rp, const float *llr, int64_t frames, int L, int T, bool early,
                    bool literal, bool loc16, float *posterior, uint8_t *bits, int32_t *iters_out, uint8_t *conv_out,
                    unsigned long long *stats, int *work_counter, cudaStream_t st) {
    (void)loc16;
    ResArgs a;
    a.g = g;
    a.llr = llr;
    a.frames = frames;
    a.L = L;
    a.T = T;
    a.early = early ? 1 : 0;
    a.literal = literal ? 1 : 0;
    a.post = posterior;
    a.bits = bits;
    a.iters = iters_out;
    a.conv = conv_out;
    a.stats = stats;
    a.counter = work_counter;
    a.rs = reinterpret_cast<float *>(reinterpret_cast<char *>(work_counter) + 256);
    a.dm = rp.dm;
    a.dc = rp.regular ? rp.dm : 0;
    a.dv = rp.regular ? rp.dv : 0;
    // LDPC_RES_GENERIC=1: no regular-code instance (rows of degree <= 8 still take the bounded-degree one);
    // =2: the any-degree instance
    a.any_degree = 0;
    if (const char *e = getenv("LDPC_RES_GENERIC")) {
        a.dc = a.dv = 0;
        a.any_degree = atoi(e) >= 2;
    }
    a.compact = rp.compact ? 1 : 0;
    a.gg = rp.global_graph ? 1 : 0;
    a.lay = layout_for(rp.slots, g.m, g.n, g.E, rp.dm, rp.compact, rp.global_graph);
    cudaMemsetAsync(work_counter, 0, sizeof(int), st);
    switch (rp.slots) {
        case 32: launch_t<32>(a, rp.threads, rp.ctas, rp.smem, st); break;
        case 16: launch_t<16>(a, rp.threads, rp.ctas, rp.smem, st); break;
        case 8: launch_t<8>(a, rp.threads, rp.ctas, rp.smem, st); break;
        default: launch_t<4>(a, rp.threads, rp.ctas, rp.smem, st); break;
    }
    return 1;
}

size_t resident_scratch_bytes(const HostGraph &g, const ResidentPlan &rp) {
    return 256 + (size_t)rp.ctas * g.n * rp.slots * 4;
}

}  // namespace ldpc
