// decode_resident.cu -- the SMEM-resident schedule: one persistent CTA per SM decodes S frames at a
// time with the whole per-frame state in shared memory, and refills a frame slot the moment its
// frame stops (per-frame early stop of Alg. 1, without batch-level waste).
//
// Per CTA, frame-interleaved over S slots (a lane owns 4 consecutive slots of one row, edge or column):
//   xe   [E][S]  fp32          lambda_e - eta_e, the check-node inputs, written by
//                              the bit-node pass so the check node never rebuilds eta^prev
//   s    [n][S]  fp32          soft vector (Eq. sCalculation)
//   min0 [m][S]  fp32          Observation 1's minimum
//   min1 [m][S]  fp32          Observation 1's second minimum
//   lc   [m][S]  u32           min0Location, stored as the edge id inside the row lists (0xffff = none)
//   par  [m]     S bits        the row's sign parity (Obs. 2) times (-1)^{d_i} (reading A1)
//   sg   [E]     S bits        sign of lambda_e - eta_e for each slot
//   hb   [n]     S bits        hard decision b_j = (s_j > 0) for the syndrome
// plus the Tanner graph itself as 16-bit lists (N_i, M_j).  r lives in a global scratch
// [CTA][n][S] (L2-resident) read once per column per body.  Loop per round:
//   A  finish stopped slots (k, isCodeword, counters) and refill empty slots from a global counter
//   B  stage new frames into their slots (s = r, x_e = r_j, hard decisions of r)
//   C  check-node pass over all rows (min0/min1/loc/parity/signs from x_e) + syndrome from hb words
//   D  per slot: stop (codeword, or k = L) -> write b and s; else bit-node pass s = sum eta + r and
//      the next x_e = s_j - eta_e (same fp32 subtraction as the oracle's lambda_k - eta^prev_{i,k})
// Every sweep uses the same lane mapping (4 slots of one row/edge/column per lane, 16-byte accesses).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "ldpc_internal.cuh"

namespace ldpc {

namespace {

constexpr unsigned FULLM = 0xffffffffu;

template <int S>
struct SWord;
template <>
struct SWord<4> {
    using T = uint8_t;
};
template <>
struct SWord<8> {
    using T = uint8_t;
};
template <>
struct SWord<16> {
    using T = uint16_t;
};
template <>
struct SWord<32> {
    using T = uint32_t;
};

struct Layout {
    size_t xe, s, m0, m1, lc, sg, par, hb, rp, cp, col, rec, meta, total;
};

constexpr size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }

constexpr int META_INTS = 8 * 32 + 16;
constexpr int DVMAX = 8;  // column degrees up to this keep their eta values in registers

Layout layout_for(int S, int m, int n, int E) {
    Layout L{};
    size_t o = 0;
    const size_t swb = S <= 8 ? 1 : S / 8;
    L.xe = o;   o = a16(o + (size_t)E * S * 4);
    L.s = o;    o = a16(o + (size_t)n * S * 4);
    L.m0 = o;   o = a16(o + (size_t)m * S * 4);
    L.m1 = o;   o = a16(o + (size_t)m * S * 4);
    L.lc = o;   o = a16(o + (size_t)m * S * 4);
    L.sg = o;   o = a16(o + (size_t)E * swb);
    L.par = o;  o = a16(o + (size_t)m * swb);
    L.hb = o;   o = a16(o + (size_t)n * swb);
    L.rp = o;   o = a16(o + (size_t)(m + 1) * 2);
    L.cp = o;   o = a16(o + (size_t)(n + 1) * 2);
    L.col = o;  o = a16(o + (size_t)E * 2);
    L.rec = o;  o = a16(o + (size_t)E * 4);
    L.meta = o; o = a16(o + (size_t)META_INTS * 4 + 8 * 8);
    L.total = o;
    return L;
}

struct ResArgs {
    Graph g;
    const float *llr;
    int64_t frames;
    int L, early, literal;
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
// min0Location test on two packed 16-bit edge ids: true iff the half selected by `hi` differs from e
__device__ __forceinline__ bool loc_ne(unsigned pair, unsigned e2, bool hi) {
    return ((pair ^ e2) & (hi ? 0xffff0000u : 0x0000ffffu)) != 0u;
}


// 32-bit shared-window addresses: the hot loops address shared memory through plain registers
// (no generic-to-shared conversion per access).
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds_u4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f4(uint32_t a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void sts_u4(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
template <int S>
__device__ __forceinline__ uint32_t lds_sw(uint32_t a) {
    return S == 32 ? lds_u32(a) : S == 16 ? lds_u16(a) : lds_u8(a);
}
template <int S>
__device__ __forceinline__ void sts_sw(uint32_t a, uint32_t v) {
    if (S == 32) asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
    else if (S == 16) asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((uint16_t)v) : "memory");
    else asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
template <int S>
constexpr int SWB() { return S <= 8 ? 1 : S / 8; }

// S-bit word of a row group from the four per-component ballots: slot q = 4l+v sits at bit v*LR + l.
template <int S>
__device__ __forceinline__ unsigned gather_word(const unsigned bal[4], int sub) {
    constexpr int LR = S / 4;
    constexpr unsigned LMASK = (LR == 32) ? 0xffffffffu : ((1u << LR) - 1u);
    unsigned word = 0;
#pragma unroll
    for (int v = 0; v < 4; v++) word |= ((bal[v] >> (sub * LR)) & LMASK) << (v * LR);
    return word;
}
// this lane's 4 slot bits (bit v = slot 4l+v) of an S-bit word
template <int S>
__device__ __forceinline__ unsigned lane_bits(unsigned word, int l) {
    constexpr int LR = S / 4;
    return ((word >> l) & 1u) | (((word >> (LR + l)) & 1u) << 1) | (((word >> (2 * LR + l)) & 1u) << 2) |
           (((word >> (3 * LR + l)) & 1u) << 3);
}


// Check-node update of one row per row group for the 4 slots of this lane, from x_e = lambda_e -
// eta^prev_e: min0 / min0Location / min1 (Obs. 1), sign parity and sign bits (Obs. 2), plus the
// row syndrome of b from the hard-decision words.  HAS: rows of the warp differ in degree.
template <int S, bool HAS>
__device__ __forceinline__ void cn_row(uint32_t SB, const Layout &lay, int i, bool valid, int ra, int d, int dmax,
                                       int l, int sub, unsigned corr_all, unsigned &syn_acc) {
    constexpr int SWBY = SWB<S>();
    const float INF = __int_as_float(0x7f800000);
    const int q0 = 4 * l;
    const uint32_t XE = SB + (uint32_t)lay.xe, SG = SB + (uint32_t)lay.sg, HB = SB + (uint32_t)lay.hb,
                   COL = SB + (uint32_t)lay.col;
    float nm0[4] = {INF, INF, INF, INF}, nm1[4] = {INF, INF, INF, INF};
    int nloc[4] = {0xffff, 0xffff, 0xffff, 0xffff};
    unsigned parw[4] = {0, 0, 0, 0};
    unsigned synw = 0;
#pragma unroll 2
    for (int p = 0; p < dmax; p++) {
        const bool has = HAS ? (p < d) : true;
        const int e = ra + p;
        float4 xv = make_float4(INF, INF, INF, INF);
        if (has) {
            xv = lds_f4(XE + (uint32_t)((e * S + q0) * 4));
            synw ^= lds_sw<S>(HB + lds_u16(COL + 2u * (uint32_t)e) * SWBY);  // b_j = slice(s_j)
        }
        unsigned bal[4];
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const float x = f4c(xv, v);
            const float ax = fabsf(x);
            const bool lt = ax < nm0[v];  // first strict minimum (A13)
            nm1[v] = fminf(nm1[v], fmaxf(nm0[v], ax));
            nm0[v] = fminf(nm0[v], ax);
            nloc[v] = lt ? e : nloc[v];
            bal[v] = __ballot_sync(FULLM, x < 0.f);  // sign(0) = +1; INF is +
        }
#pragma unroll
        for (int v = 0; v < 4; v++) parw[v] ^= bal[v];
        if (has && l == 0) sts_sw<S>(SG + (uint32_t)(e * SWBY), gather_word<S>(bal, sub));
    }
    if (valid) {
        const uint32_t ca = (uint32_t)((i * S + q0) * 4);
        sts_f4(SB + (uint32_t)lay.m0 + ca, make_float4(nm0[0], nm0[1], nm0[2], nm0[3]));
        sts_f4(SB + (uint32_t)lay.m1 + ca, make_float4(nm1[0], nm1[1], nm1[2], nm1[3]));
        sts_u4(SB + (uint32_t)lay.lc + ca, make_uint4(nloc[0], nloc[1], nloc[2], nloc[3]));
        if (l == 0)
            sts_sw<S>(SB + (uint32_t)lay.par + (uint32_t)(i * SWBY),
                      gather_word<S>(parw, sub) ^ ((d & 1) ? corr_all : 0u));  // (-1)^{d_i}, reading A1
        syn_acc |= lane_bits<S>(synw, l);
    }
}

// eta_{i,j} of one column edge (record rc = e << 16 | i) for the 4 slots of this lane (Obs. 1/2)
template <int S>
__device__ __forceinline__ void eta_of(uint32_t SB, const Layout &lay, uint32_t rc, int q0, const unsigned mv[4],
                                       float et[4]) {
    constexpr int SWBY = SWB<S>();
    const int e = (int)(rc >> 16), i = (int)(rc & 0xffffu);
    const uint32_t ca = (uint32_t)((i * S + q0) * 4);
    const float4 m0 = lds_f4(SB + (uint32_t)lay.m0 + ca);
    const float4 m1 = lds_f4(SB + (uint32_t)lay.m1 + ca);
    const uint4 lv = lds_u4(SB + (uint32_t)lay.lc + ca);
    const unsigned W = lds_sw<S>(SB + (uint32_t)lay.sg + (uint32_t)(e * SWBY)) ^
                       lds_sw<S>(SB + (uint32_t)lay.par + (uint32_t)(i * SWBY));
    const float mg0 = ((int)lv.x == e) ? m1.x : m0.x;
    const float mg1 = ((int)lv.y == e) ? m1.y : m0.y;
    const float mg2 = ((int)lv.z == e) ? m1.z : m0.z;
    const float mg3 = ((int)lv.w == e) ? m1.w : m0.w;
    et[0] = (W & mv[0]) ? -mg0 : mg0;
    et[1] = (W & mv[1]) ? -mg1 : mg1;
    et[2] = (W & mv[2]) ? -mg2 : mg2;
    et[3] = (W & mv[3]) ? -mg3 : mg3;
}

// Lane layout: a lane owns 4 consecutive slots (float4) of one row, edge or column; LR = S/4 lanes
// cover a row, G = 32/LR rows per warp.  Bit of slot q = 4*l + v inside an S-bit word: v*LR + l.
template <int S, int RT>
__global__ void __launch_bounds__(RT, 1) k_resident(ResArgs a) {
    constexpr int NWARP = RT / 32;
    using SWT = typename SWord<S>::T;
    constexpr int LR = S / 4;
    constexpr int G = 32 / LR;
    extern __shared__ __align__(16) unsigned char sm[];
    const int m = a.g.m, n = a.g.n, E = a.g.E;
    float *xe = reinterpret_cast<float *>(sm + a.lay.xe);
    float *s = reinterpret_cast<float *>(sm + a.lay.s);
    float *mn0 = reinterpret_cast<float *>(sm + a.lay.m0);
    float *mn1 = reinterpret_cast<float *>(sm + a.lay.m1);
    SWT *sg = reinterpret_cast<SWT *>(sm + a.lay.sg);
    SWT *par = reinterpret_cast<SWT *>(sm + a.lay.par);
    SWT *hb = reinterpret_cast<SWT *>(sm + a.lay.hb);
    uint16_t *rp = reinterpret_cast<uint16_t *>(sm + a.lay.rp);
    uint16_t *cp = reinterpret_cast<uint16_t *>(sm + a.lay.cp);
    uint16_t *col = reinterpret_cast<uint16_t *>(sm + a.lay.col);
    uint32_t *rec = reinterpret_cast<uint32_t *>(sm + a.lay.rec);
    int *meta = reinterpret_cast<int *>(sm + a.lay.meta);
    int *slot_f = meta;            // frame index of the slot, -1 = empty
    int *slot_k = meta + 32;       // completed loop bodies
    int *slot_be = meta + 64;      // ones of b (bit errors vs the all-zero codeword)
    int *slot_raw = meta + 96;     // r_j > 0 count
    int *slot_nz = meta + 128;     // some |s_j| <= 1e-4
    unsigned *ctl = reinterpret_cast<unsigned *>(meta + 256);  // [0] unsat, [1] new, [2] active, [3] exhausted

    const uint32_t SB = smem_u32(sm);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sub = lane / LR, l = lane % LR;  // row group inside the warp, lane inside the row
    const int q0 = 4 * l;                      // first slot of this lane
    float *rs = a.rs + (size_t)blockIdx.x * n * S;
    const unsigned corr_all = a.literal ? 0u : (S == 32 ? 0xffffffffu : ((1u << S) - 1u));

    // ---- the Tanner graph into shared memory (16-bit lists)
    for (int q = tid; q <= m; q += RT) rp[q] = (uint16_t)__ldg(a.g.row_ptr + q);
    for (int q = tid; q <= n; q += RT) cp[q] = (uint16_t)__ldg(a.g.col_ptr + q);
    for (int e = tid; e < E; e += RT) {
        col[e] = (uint16_t)__ldg(a.g.col_idx + e);
        const int4 be = __ldg(a.g.bn_edge + e);  // {edge id, row, pos, parity}
        rec[e] = ((uint32_t)be.x << 16) | (uint32_t)be.y;
    }
    if (tid < 32) {
        slot_f[tid] = -1;
        slot_k[tid] = 0;
        slot_be[tid] = 0;
        slot_raw[tid] = 0;
        slot_nz[tid] = 0;
    }
    if (tid == 0) {
        ctl[0] = 0;
        ctl[1] = 0;
        ctl[2] = 0;
        ctl[3] = 0;
    }
    unsigned long long acc_stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // warp 0, lane = slot
    unsigned mv[4];
#pragma unroll
    for (int v = 0; v < 4; v++) mv[v] = 1u << (v * LR + l);
    __syncthreads();

    for (;;) {
        // ---------------- A: finish stopped slots, advance continuing ones, refill (warp 0)
        if (warp == 0) {
            const unsigned uns_all = ctl[0];
            const unsigned act_all = ctl[2];
            const bool mine = lane < S;
            int f = mine ? slot_f[lane] : 0;
            if (mine && ((act_all >> lane) & 1u)) {
                const int k = slot_k[lane];
                const bool uns = (uns_all >> lane) & 1u;
                const bool fin = a.early ? (!uns || k == a.L) : (k == a.L);
                if (fin) {
                    const int conv = !uns;
                    if (a.iters) a.iters[f] = k;
                    if (a.conv) a.conv[f] = (uint8_t)conv;
                    const int be = slot_be[lane];
                    acc_stats[0] += 1;
                    acc_stats[1] += (unsigned long long)be;
                    acc_stats[2] += be > 0;
                    acc_stats[3] += (be > 0) && conv;
                    acc_stats[4] += (unsigned long long)k;
                    acc_stats[5] += conv;
                    acc_stats[6] += slot_nz[lane] != 0;
                    acc_stats[7] += (unsigned long long)slot_raw[lane];
                    f = -1;
                } else {
                    slot_k[lane] = k + 1;
                }
            }
            // refill: the free slots take consecutive frames from the global counter
            const unsigned freem = __ballot_sync(FULLM, mine && f < 0);
            long long base = 0;
            if (lane == 0 && freem && !ctl[3]) base = atomicAdd(a.counter, __popc(freem));
            base = __shfl_sync(FULLM, base, 0);
            const bool exhausted = ctl[3] != 0;
            unsigned fresh = 0;
            if (freem && !exhausted) {
                const long long mine_f = base + __popc(freem & ((1u << lane) - 1u));
                const bool take = mine && f < 0 && mine_f < a.frames;
                if (take) {
                    f = (int)mine_f;
                    slot_k[lane] = 0;
                    slot_be[lane] = 0;
                    slot_raw[lane] = 0;
                    slot_nz[lane] = 0;
                }
                fresh = __ballot_sync(FULLM, take);
                if (lane == 0 && base + __popc(freem) >= a.frames) ctl[3] = 1;
            }
            if (mine) slot_f[lane] = f;
            const unsigned active = __ballot_sync(FULLM, mine && f >= 0);
            if (lane == 0) {
                ctl[0] = 0;
                ctl[1] = fresh;
                ctl[2] = active;
            }
        }
        __syncthreads();
        const unsigned active = ctl[2], fresh_new = ctl[1];
        if (!active) break;

        // ---------------- B: stage new frames: s = r, lambda_e - eta_e = r (eta = 0),
        //                     hard decisions of r for the pre-loop test
        if (fresh_new) {
            const unsigned fm = (fresh_new >> q0) & 0xfu;  // this lane's fresh slots
            SWT fw = 0;                                     // S-bit word of the fresh slots
#pragma unroll
            for (int q = 0; q < S; q++)
                if ((fresh_new >> q) & 1u) fw |= (SWT)(1u << ((q & 3) * LR + (q >> 2)));
            int fr[4];
#pragma unroll
            for (int v = 0; v < 4; v++) fr[v] = slot_f[q0 + v];
            int raw[4] = {0, 0, 0, 0};
            for (int cb = warp * G; cb < n; cb += NWARP * G) {
                const int j = cb + sub;
                const bool jv = j < n;
                float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                if (jv && fm) {
                    float *sp = s + j * S + q0;
                    o = *reinterpret_cast<const float4 *>(sp);
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        if ((fm >> v) & 1u) {
                            const float x = __ldg(a.llr + (int64_t)fr[v] * n + j);
                            f4s(o, v, x);
                            rs[(size_t)j * S + q0 + v] = x;
                            raw[v] += x > 0.f;
                        }
                    }
                    *reinterpret_cast<float4 *>(sp) = o;
                    const int c0 = cp[j], dv = (int)cp[j + 1] - c0;
                    for (int qq = 0; qq < dv; qq++) {
                        const int e = (int)(rec[c0 + qq] >> 16);
                        float *xp = xe + e * S + q0;
                        float4 xo = *reinterpret_cast<const float4 *>(xp);
#pragma unroll
                        for (int v = 0; v < 4; v++)
                            if ((fm >> v) & 1u) f4s(xo, v, f4c(o, v));
                        *reinterpret_cast<float4 *>(xp) = xo;
                    }
                }
                unsigned bal[4];
#pragma unroll
                for (int v = 0; v < 4; v++) bal[v] = __ballot_sync(FULLM, jv && f4c(o, v) > 0.f);
                if (jv && l == 0) hb[j] = (SWT)(((unsigned)hb[j] & ~(unsigned)fw) | (gather_word<S>(bal, sub) & fw));
            }
#pragma unroll
            for (int v = 0; v < 4; v++) {
                int x = raw[v];
                for (int o = LR; o < 32; o <<= 1) x += __shfl_xor_sync(FULLM, x, o);
                if (sub == 0 && x) atomicAdd(&slot_raw[q0 + v], x);
            }
            __syncthreads();
        }

        // ---------------- C: check-node pass over x_e = s_j - eta^prev_e + syndrome of b
        {
            unsigned syn_acc = 0;  // bit v: slot q0+v has an unsatisfied check
            for (int rb = warp * G; rb < m; rb += NWARP * G) {
                const int i = rb + sub;
                const bool valid = i < m;
                const int ra = valid ? rp[i] : 0;
                const int d = valid ? (int)rp[i + 1] - ra : 0;
                const int dmax = __reduce_max_sync(FULLM, d);
                if (__all_sync(FULLM, d == dmax))
                    cn_row<S, false>(SB, a.lay, i, valid, ra, d, dmax, l, sub, corr_all, syn_acc);
                else
                    cn_row<S, true>(SB, a.lay, i, valid, ra, d, dmax, l, sub, corr_all, syn_acc);
            }
            const unsigned mine = (syn_acc << q0) & active;
            const unsigned wmask = __reduce_or_sync(FULLM, mine);
            if (lane == 0 && wmask) atomicOr(&ctl[0], wmask);
        }
        __syncthreads();

        // ---------------- D: per-slot decision; outputs of stopping slots and the bit-node update
        //                     (Eq. lambda_j) of the continuing ones in one column sweep
        {
            const unsigned uns_all = ctl[0];
            bool fin = false, cont = false;
            if (lane < S && ((active >> lane) & 1u)) {
                const int k = slot_k[lane];
                const bool uns = (uns_all >> lane) & 1u;
                fin = a.early ? (!uns || k == a.L) : (k == a.L);
                cont = !fin;
            }
            const unsigned fin_mask = __ballot_sync(FULLM, fin), cont_mask = __ballot_sync(FULLM, cont);
            const unsigned cm = (cont_mask >> q0) & 0xfu;  // continuing slots of this lane
            const unsigned fk = (fin_mask >> q0) & 0xfu;   // stopping slots of this lane
            if (fin_mask | cont_mask) {
                int64_t fo[4];
#pragma unroll
                for (int v = 0; v < 4; v++) fo[v] = (int64_t)slot_f[q0 + v] * n;
                int be[4] = {0, 0, 0, 0};
                unsigned nz = 0;
                for (int cb = warp * G; cb < n; cb += NWARP * G) {
                    const int j = cb + sub;
                    const bool jv = j < n;
                    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (jv && fk) {
                        o = *reinterpret_cast<const float4 *>(s + j * S + q0);
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
                    const bool work = jv && cm;
                    if (work) {
                        const float4 rj = *reinterpret_cast<const float4 *>(rs + (size_t)j * S + q0);
                        const int c0 = cp[j], dv = (int)cp[j + 1] - c0;
                        float acc[4] = {0.f, 0.f, 0.f, 0.f};
                        float eta[DVMAX][4];
                        int ee[DVMAX];
#pragma unroll
                        for (int qq = 0; qq < DVMAX; qq++) {
                            if (qq < dv) {
                                const uint32_t rc = rec[c0 + qq];
                                ee[qq] = (int)(rc >> 16);
                                eta_of<S>(SB, a.lay, rc, q0, mv, eta[qq]);
#pragma unroll
                                for (int v = 0; v < 4; v++) acc[v] = acc[v] + eta[qq][v];  // ascending rows (A14)
                            }
                        }
                        for (int qq = DVMAX; qq < dv; qq++) {
                            float et[4];
                            eta_of<S>(SB, a.lay, rec[c0 + qq], q0, mv, et);
#pragma unroll
                            for (int v = 0; v < 4; v++) acc[v] = acc[v] + et[v];
                        }
                        float4 sn = make_float4(acc[0] + rj.x, acc[1] + rj.y, acc[2] + rj.z, acc[3] + rj.w);
                        sts_f4(SB + (uint32_t)a.lay.s + (uint32_t)((j * S + q0) * 4), sn);
                        // extrinsic values for the next check-node pass: x_e = s_j - eta_e
#pragma unroll
                        for (int qq = 0; qq < DVMAX; qq++) {
                            if (qq < dv)
                                sts_f4(SB + (uint32_t)a.lay.xe + (uint32_t)((ee[qq] * S + q0) * 4),
                                       make_float4(sn.x - eta[qq][0], sn.y - eta[qq][1], sn.z - eta[qq][2],
                                                   sn.w - eta[qq][3]));
                        }
                        for (int qq = DVMAX; qq < dv; qq++) {
                            const uint32_t rc = rec[c0 + qq];
                            float et[4];
                            eta_of<S>(SB, a.lay, rc, q0, mv, et);
                            sts_f4(SB + (uint32_t)a.lay.xe + (uint32_t)(((int)(rc >> 16) * S + q0) * 4),
                                   make_float4(sn.x - et[0], sn.y - et[1], sn.z - et[2], sn.w - et[3]));
                        }
                        o = sn;
                    }
                    // hard decisions of the new s for the next syndrome (continuing slots only matter)
                    unsigned bal[4];
#pragma unroll
                    for (int v = 0; v < 4; v++) bal[v] = __ballot_sync(FULLM, work && f4c(o, v) > 0.f);
                    if (jv && l == 0 && cont_mask) hb[j] = (SWT)gather_word<S>(bal, sub);
                }
                if (fin_mask) {
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        int x = be[v];
                        for (int o = LR; o < 32; o <<= 1) x += __shfl_xor_sync(FULLM, x, o);
                        if (sub == 0 && x) atomicAdd(&slot_be[q0 + v], x);
                    }
                    unsigned z = nz;
                    for (int o = LR; o < 32; o <<= 1) z |= __shfl_xor_sync(FULLM, z, o);
                    if (sub == 0 && z)
#pragma unroll
                        for (int v = 0; v < 4; v++)
                            if ((z >> v) & 1u) slot_nz[q0 + v] = 1;
                }
            }
        }
        __syncthreads();
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

template <int S, int RT>
void launch_s(const ResArgs &args, int ctas, size_t smem, cudaStream_t st) {
    cudaFuncSetAttribute(k_resident<S, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_resident<S, RT><<<ctas, RT, smem, st>>>(args);
}

template <int S>
void launch_t(const ResArgs &args, int threads, int ctas, size_t smem, cudaStream_t st) {
    if (threads == 1024) launch_s<S, 1024>(args, ctas, smem, st);
    else if (threads == 768) launch_s<S, 768>(args, ctas, smem, st);
    else launch_s<S, 512>(args, ctas, smem, st);
}

}  // namespace

ResidentPlan plan_resident(const HostGraph &g, bool loc16, int device) {
    (void)loc16;
    ResidentPlan rp;
    if (g.n >= 65535 || g.m >= 65535 || g.E >= 65535 || g.E == 0) return rp;
    const int cap = max_smem_optin(device);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (cap <= 0 || sms <= 0) return rp;
    for (int S : {32, 16, 8, 4}) {
        const Layout L = layout_for(S, g.m, g.n, g.E);
        if (L.total <= (size_t)cap) {
            rp.ok = true;
            rp.slots = S;
            rp.threads = 512;
            if (const char *e = getenv("LDPC_RES_THREADS")) {
                const int t = atoi(e);
                rp.threads = (t == 1024 || t == 768) ? t : 512;
            }
            rp.smem = L.total;
            rp.ctas = sms;
            return rp;
        }
    }
    return rp;
}

// rs scratch is carved after the two counter ints of work_counter's allocation owner (runtime.cu)
int launch_resident(const Graph &g, const ResidentPlan &rp, const float *llr, int64_t frames, int L, bool early,
                    bool literal, bool loc16, float *posterior, uint8_t *bits, int32_t *iters_out, uint8_t *conv_out,
                    unsigned long long *stats, int *work_counter, cudaStream_t st) {
    (void)loc16;
    ResArgs a;
    a.g = g;
    a.llr = llr;
    a.frames = frames;
    a.L = L;
    a.early = early ? 1 : 0;
    a.literal = literal ? 1 : 0;
    a.post = posterior;
    a.bits = bits;
    a.iters = iters_out;
    a.conv = conv_out;
    a.stats = stats;
    a.counter = work_counter;
    a.rs = reinterpret_cast<float *>(reinterpret_cast<char *>(work_counter) + 256);
    a.lay = layout_for(rp.slots, g.m, g.n, g.E);
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
