// decode_resident.cu -- the SMEM-resident schedule: one persistent CTA per SM decodes S frames at a
// time with the whole per-frame state in shared memory, and refills a frame slot the moment its
// frame stops (per-frame early stop of Alg. 1, without batch-level waste).
//
// Per CTA, frame-interleaved over S slots (a lane owns 4 consecutive slots of one row, edge or column):
//   xe [E][S] fp32   the per-edge message of the paper's map-reduce form (Alg. 2) restricted
//                    to the edges of H: it holds lambda(i,j) = s(j) - eta(i,j) before the
//                    check-node pass and eta(i,j) (Eq. etaCalculation) after it
//   hb [n]    S bits hard decision b_j = (s_j > 0) (Eq. slice) for the syndrome
// plus the Tanner graph as 16-bit lists (N_i, M_j).  r and the soft vector s (Eq. sCalculation,
// P:337-344) live in L2-resident global scratch [CTA][n][S]: the check node never reads s (it reads
// lambda), so s is only written by the column sums and read back for the output.  Loop per round:
//   A  finish stopped slots (k, isCodeword, counters) and refill empty slots from a global counter
//   B  stage new frames into their slots (s = r, lambda = r on every edge, hard decisions of r)
//   C  check-node pass over all rows: reduce lambda to min0/min0Location/min1/parity (Obs. 1/2), then
//      write eta in place; the same pass XORs the hard decisions of the row into the syndrome
//   D  per slot: stop (codeword, or k = L) -> write b and s; else column sums s = sum eta + r and the
//      next lambda = s - eta (fp32, ascending rows from +0.0 then + r, reading A14)
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
    size_t xe, hb, rp, cp, col, ce, meta, total;
};

constexpr size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }

constexpr int META_INTS = 8 * 32 + 16;

Layout layout_for(int S, int m, int n, int E) {
    Layout L{};
    size_t o = 0;
    const size_t swb = S <= 8 ? 1 : S / 8;
    L.xe = o;   o = a16(o + (size_t)E * S * 4);
    L.hb = o;   o = a16(o + (size_t)n * swb);
    L.rp = o;   o = a16(o + (size_t)(m + 1) * 2);
    L.cp = o;   o = a16(o + (size_t)(n + 1) * 2);
    L.col = o;  o = a16(o + (size_t)E * 2);
    L.ce = o;   o = a16(o + (size_t)E * 2);
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
    float *rs;  // [CTA][n][S] channel values r of the slots (global, L2-resident)
    float *ss;  // [CTA][n][S] soft vectors s of the slots (global, L2-resident)
    Layout lay;
};

__device__ __forceinline__ float f4c(const float4 &a, int v) { return v == 0 ? a.x : v == 1 ? a.y : v == 2 ? a.z : a.w; }
__device__ __forceinline__ void f4s(float4 &a, int v, float x) {
    if (v == 0) a.x = x;
    else if (v == 1) a.y = x;
    else if (v == 2) a.z = x;
    else a.w = x;
}

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

// Check-node update of one row per row group for the 4 slots of this lane (Eq. etaCalculation,
// P:327-336).  Pass 1 reduces lambda(i,j) of the row to min0, min0Location, min1 (Obs. 1) and the sign
// parity (Obs. 2) -- the paper's four vectors -- and XORs the row's hard decisions into the
// syndrome.  Pass 2 overwrites lambda(i,j) with eta(i,j) in place.  HAS: rows of the warp differ in degree.
template <int S, bool HAS>
__device__ __forceinline__ void cn_row(float *xe, const uint16_t *col, const typename SWord<S>::T *hb, int i,
                                       bool valid, int ra, int xb, int d, int dmax, int l, int lane,
                                       bool corr_lit, unsigned &syn_acc) {
    constexpr int DR = 8;  // row degrees up to DR keep lambda in registers between the two passes
    const float INF = __int_as_float(0x7f800000);
    const int q0 = 4 * l;
    float nm0[4] = {INF, INF, INF, INF}, nm1[4] = {INF, INF, INF, INF};
    int nloc[4] = {-1, -1, -1, -1};
    unsigned parw[4] = {0, 0, 0, 0};
    unsigned synw = 0;
    float4 xr[DR];
    auto scan = [&](int p, float4 xv) {
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const float x = f4c(xv, v);
            const float ax = fabsf(x);
            const bool lt = ax < nm0[v];  // first strict minimum (A13)
            nm1[v] = fminf(nm1[v], fmaxf(nm0[v], ax));
            nm0[v] = fminf(nm0[v], ax);
            nloc[v] = lt ? p : nloc[v];
            parw[v] ^= __ballot_sync(FULLM, x < 0.f);  // sign(0) = +1; INF is +
        }
    };
    const bool small = dmax <= DR;
    if (small) {
#pragma unroll
        for (int p = 0; p < DR; p++) {
            if (p < dmax) {
                const bool has = HAS ? (p < d) : true;
                xr[p] = make_float4(INF, INF, INF, INF);
                if (has) {
                    xr[p] = *reinterpret_cast<const float4 *>(xe + (xb + p) * S + q0);
                    synw ^= (unsigned)hb[col[ra + p]];  // b_j = slice(s_j)
                }
                scan(p, xr[p]);
            }
        }
    } else {
        for (int p = 0; p < dmax; p++) {
            const bool has = HAS ? (p < d) : true;
            float4 xv = make_float4(INF, INF, INF, INF);
            if (has) {
                xv = *reinterpret_cast<const float4 *>(xe + (xb + p) * S + q0);
                synw ^= (unsigned)hb[col[ra + p]];
            }
            scan(p, xv);
        }
    }
    if (valid) {
        // row parity of this lane's slots, times (-1)^{d_i} (reading A1)
        const unsigned flip = (corr_lit && (d & 1)) ? 1u : 0u;
        unsigned pv[4];
#pragma unroll
        for (int v = 0; v < 4; v++) pv[v] = ((parw[v] >> lane) & 1u) ^ flip;
        auto emit = [&](int p, float4 xv) {
            float4 o;
#pragma unroll
            for (int v = 0; v < 4; v++) {
                const float x = f4c(xv, v);
                const float mag = (p == nloc[v]) ? nm1[v] : nm0[v];       // Obs. 1 (delta placement, A2)
                const bool neg = ((unsigned)(x < 0.f) ^ pv[v]) != 0u;    // Obs. 2: parity x own sign
                f4s(o, v, neg ? -mag : mag);
            }
            *reinterpret_cast<float4 *>(xe + (xb + p) * S + q0) = o;
        };
        if (small) {
#pragma unroll
            for (int p = 0; p < DR; p++)
                if (p < d) emit(p, xr[p]);
        } else {
            for (int p = 0; p < d; p++) emit(p, *reinterpret_cast<const float4 *>(xe + (xb + p) * S + q0));
        }
        syn_acc |= lane_bits<S>(synw, l);
    }
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
    SWT *hb = reinterpret_cast<SWT *>(sm + a.lay.hb);
    uint16_t *rp = reinterpret_cast<uint16_t *>(sm + a.lay.rp);
    uint16_t *cp = reinterpret_cast<uint16_t *>(sm + a.lay.cp);
    uint16_t *col = reinterpret_cast<uint16_t *>(sm + a.lay.col);
    uint16_t *ce = reinterpret_cast<uint16_t *>(sm + a.lay.ce);
    int *meta = reinterpret_cast<int *>(sm + a.lay.meta);
    int *slot_f = meta;            // frame index of the slot, -1 = empty
    int *slot_k = meta + 32;       // completed loop bodies
    int *slot_be = meta + 64;      // ones of b (bit errors vs the all-zero codeword)
    int *slot_raw = meta + 96;     // r_j > 0 count
    int *slot_nz = meta + 128;     // some |s_j| <= 1e-4
    unsigned *ctl = reinterpret_cast<unsigned *>(meta + 256);  // [0] unsat, [1] new, [2] active, [3] exhausted

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sub = lane / LR, l = lane % LR;  // row group inside the warp, lane inside the row
    const int q0 = 4 * l;                      // first slot of this lane
    float *rs = a.rs + (size_t)blockIdx.x * n * S;
    float *ssg = a.ss + (size_t)blockIdx.x * n * S;
    const bool corr = !a.literal;

    // ---- the Tanner graph into shared memory (16-bit lists)
    for (int q = tid; q <= m; q += RT) rp[q] = (uint16_t)__ldg(a.g.row_ptr + q);
    for (int q = tid; q <= n; q += RT) cp[q] = (uint16_t)__ldg(a.g.col_ptr + q);
    for (int e = tid; e < E; e += RT) col[e] = (uint16_t)__ldg(a.g.col_idx + e);
    for (int q = tid; q < E; q += RT) ce[q] = (uint16_t)__ldg(&a.g.bn_edge[q].x);  // M_j as edge ids
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

        // ---------------- B: stage new frames: s = r and lambda(i,j) = r(j) on every edge (eta = 0,
        //                     P:124-127), hard decisions of r for the pre-loop test
        if (fresh_new) {
            const unsigned fm = (fresh_new >> q0) & 0xfu;  // this lane's fresh slots
            unsigned fw = 0;                                // S-bit word of the fresh slots
#pragma unroll
            for (int q = 0; q < S; q++)
                if ((fresh_new >> q) & 1u) fw |= 1u << ((q & 3) * LR + (q >> 2));
            int fr[4];
#pragma unroll
            for (int v = 0; v < 4; v++) fr[v] = slot_f[q0 + v];
            int raw[4] = {0, 0, 0, 0};
            for (int cb = warp * G; cb < n; cb += NWARP * G) {
                const int j = cb + sub;
                const bool jv = j < n;
                float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                if (jv && fm) {
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        if ((fm >> v) & 1u) {
                            const float x = __ldg(a.llr + (int64_t)fr[v] * n + j);
                            f4s(o, v, x);
                            rs[(size_t)j * S + q0 + v] = x;
                            ssg[(size_t)j * S + q0 + v] = x;
                            raw[v] += x > 0.f;
                        }
                    }
                    const int c0 = cp[j], dv = (int)cp[j + 1] - c0;
                    for (int qq = 0; qq < dv; qq++) {
                        float *xp = xe + (int)ce[c0 + qq] * S + q0;
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
                if (jv && l == 0) hb[j] = (SWT)(((unsigned)hb[j] & ~fw) | (gather_word<S>(bal, sub) & fw));
            }
#pragma unroll
            for (int v = 0; v < 4; v++) {
                int x = raw[v];
                for (int o = LR; o < 32; o <<= 1) x += __shfl_xor_sync(FULLM, x, o);
                if (sub == 0 && x) atomicAdd(&slot_raw[q0 + v], x);
            }
            __syncthreads();
        }

        // ---------------- C: check-node pass: lambda -> eta on every edge + syndrome of b
        {
            unsigned syn_acc = 0;  // bit v: slot q0+v has an unsatisfied check
            for (int rb = warp * G; rb < m; rb += NWARP * G) {
                const int i = rb + sub;
                const bool valid = i < m;
                const int ra = valid ? rp[i] : 0;
                const int d = valid ? (int)rp[i + 1] - ra : 0;
                const int dmax = __reduce_max_sync(FULLM, d);
                if (__all_sync(FULLM, d == dmax))
                    cn_row<S, false>(xe, col, hb, i, valid, ra, ra, d, dmax, l, lane, corr, syn_acc);
                else
                    cn_row<S, true>(xe, col, hb, i, valid, ra, ra, d, dmax, l, lane, corr, syn_acc);
            }
            const unsigned mine = (syn_acc << q0) & active;
            const unsigned wmask = __reduce_or_sync(FULLM, mine);
            if (lane == 0 && wmask) atomicOr(&ctl[0], wmask);
        }
        __syncthreads();

        // ---------------- D: per-slot decision; outputs of stopping slots and, for the continuing
        //                     ones, the column sums s_j = sum eta + r (Eq. sCalculation) and
        //                     the next lambda(i,j) = s(j) - eta(i,j) in one column sweep
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
                        o = *reinterpret_cast<const float4 *>(ssg + (size_t)j * S + q0);
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
                        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
                        for (int qq = 0; qq < dv; qq++) {
                            const float4 et = *reinterpret_cast<const float4 *>(xe + (int)ce[c0 + qq] * S + q0);
                            acc.x = acc.x + et.x;  // ascending rows from +0.0 (A14)
                            acc.y = acc.y + et.y;
                            acc.z = acc.z + et.z;
                            acc.w = acc.w + et.w;
                        }
                        const float4 sn = make_float4(acc.x + rj.x, acc.y + rj.y, acc.z + rj.z, acc.w + rj.w);
                        *reinterpret_cast<float4 *>(ssg + (size_t)j * S + q0) = sn;
#pragma unroll 4
                        for (int qq = 0; qq < dv; qq++) {
                            float *xp = xe + (int)ce[c0 + qq] * S + q0;
                            const float4 et = *reinterpret_cast<const float4 *>(xp);
                            *reinterpret_cast<float4 *>(xp) =
                                make_float4(sn.x - et.x, sn.y - et.y, sn.z - et.z, sn.w - et.w);
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
    if (g.n >= 65535 || g.m >= 65535 || (int64_t)g.E + g.m >= 65535 || g.E == 0) return rp;
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
    a.ss = a.rs + (size_t)rp.ctas * g.n * rp.slots;
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
    return 256 + 2 * (size_t)rp.ctas * g.n * rp.slots * 4;
}

}  // namespace ldpc
