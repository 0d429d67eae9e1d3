// decode_resident.cu -- the SMEM-resident schedule: one persistent CTA per SM decodes S frames at a
// time with the whole per-frame state in shared memory, and refills a frame slot the moment its
// frame stops (per-frame early stop of Alg. 1, without batch-level waste).
//
// Per CTA, frame-interleaved over S slots (lane l of a warp owns slot l % S of row/column l / S):
//   s   [n][S]  fp32           soft vector (Eq. sCalculation)
//   st  [m][S]  {min0, min1}   Observation 1's minima; min0's sign bit holds the row's
//                              sign parity (Obs. 2) times (-1)^{d_i} (reading A1)
//   lc  [m][S]  u16            min0Location, stored as the edge id inside the row list
//   sg  [E]     S bits         sign of lambda_e = s_j - eta_e for each slot
// plus the Tanner graph itself as 16-bit lists (N_i, M_j).  r lives in a global scratch
// [CTA][n][S] (L2-resident) read once per column per body.  Loop per round:
//   A  finish stopped slots (k, isCodeword, counters) and refill empty slots from a global counter
//   B  stage new frames into their slots (s = r, eta = 0 via k = 0)
//   C  check-node pass over all rows + syndrome of b = slice(s) of every slot
//   D  per slot: stop (codeword, or k = L) -> write b and s; else bit-node pass s = sum eta + r
#include <cuda_runtime.h>

#include <algorithm>

#include "ldpc_internal.cuh"

namespace ldpc {

namespace {

constexpr int RT = 1024;  // threads per resident CTA (32 warps)
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
    size_t s, st, lc, sg, rp, cp, col, rec, meta, total;
};

constexpr size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }

constexpr int META_INTS = 8 * 32 + 16;

Layout layout_for(int S, int m, int n, int E) {
    Layout L{};
    size_t o = 0;
    const size_t swb = S <= 8 ? 1 : S / 8;
    L.s = o;    o = a16(o + (size_t)n * S * 4);
    L.st = o;   o = a16(o + (size_t)m * S * 8);
    L.lc = o;   o = a16(o + (size_t)m * S * 2);
    L.sg = o;   o = a16(o + (size_t)E * swb);
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

template <int S>
__global__ void __launch_bounds__(RT, 1) k_resident(ResArgs a) {
    using SWT = typename SWord<S>::T;
    constexpr int G = 32 / S;  // rows (or columns) per warp
    extern __shared__ __align__(16) unsigned char sm[];
    const int m = a.g.m, n = a.g.n, E = a.g.E;
    float *s = reinterpret_cast<float *>(sm + a.lay.s);
    float2 *st = reinterpret_cast<float2 *>(sm + a.lay.st);
    uint16_t *lc = reinterpret_cast<uint16_t *>(sm + a.lay.lc);
    SWT *sg = reinterpret_cast<SWT *>(sm + a.lay.sg);
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

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sub = lane / S, slot = lane % S;
    float *rs = a.rs + (size_t)blockIdx.x * n * S;

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
    __syncthreads();

    for (;;) {
        // ---------------- A: finish stopped slots, advance continuing ones, refill (warp 0)
        if (warp == 0) {
            const unsigned uns_all = ctl[0];
            const unsigned act_all = ctl[2];
            if (lane < S && ((act_all >> lane) & 1u)) {
                const int k = slot_k[lane];
                const bool uns = (uns_all >> lane) & 1u;
                const bool fin = a.early ? (!uns || k == a.L) : (k == a.L);
                if (fin) {
                    const int64_t f = slot_f[lane];
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
                    slot_f[lane] = -1;
                } else {
                    slot_k[lane] = k + 1;
                }
            }
            __syncwarp();
            if (lane == 0) {
                ctl[0] = 0;
                unsigned fresh = 0, active = 0;
                int nfree = 0;
                for (int q = 0; q < S; q++) nfree += slot_f[q] < 0;
                if (nfree && !ctl[3]) {
                    long long base = atomicAdd(a.counter, nfree);
                    for (int q = 0; q < S; q++) {
                        if (slot_f[q] >= 0) continue;
                        if (base < a.frames) {
                            slot_f[q] = (int)base++;
                            slot_k[q] = 0;
                            slot_be[q] = 0;
                            slot_raw[q] = 0;
                            slot_nz[q] = 0;
                            fresh |= 1u << q;
                        }
                    }
                    if (base >= a.frames) ctl[3] = 1;
                }
                for (int q = 0; q < S; q++) active |= (unsigned)(slot_f[q] >= 0) << q;
                ctl[1] = fresh;
                ctl[2] = active;
            }
        }
        __syncthreads();
        const unsigned active = ctl[2], fresh_new = ctl[1];
        if (!active) break;

        // ---------------- B: stage new frames (s = r; k = 0 means eta^prev = 0)
        if (fresh_new) {
            for (unsigned fm = fresh_new; fm; fm &= fm - 1) {
                const int q = __ffs(fm) - 1;
                const float *src = a.llr + (int64_t)slot_f[q] * n;
                int raw = 0;
                for (int j = tid; j < n; j += RT) {
                    const float v = __ldg(src + j);
                    s[j * S + q] = v;
                    rs[(size_t)j * S + q] = v;
                    raw += v > 0.f;
                }
                for (int o = 16; o; o >>= 1) raw += __shfl_xor_sync(FULLM, raw, o);
                if (lane == 0 && raw) atomicAdd(&slot_raw[q], raw);
            }
            __syncthreads();
        }

        // ---------------- C: check-node pass + syndrome
        {
            const bool lane_act = (active >> slot) & 1u;
            const bool fresh = slot_k[slot] == 0;
            unsigned usyn = 0;
            for (int rb = warp * G; rb < m; rb += 32 * G) {
                const int i = rb + sub;
                const bool valid = i < m;
                const int ra = valid ? rp[i] : 0;
                const int d = valid ? (int)rp[i + 1] - ra : 0;
                const int dmax = __reduce_max_sync(FULLM, d);
                float m0 = 0.f, m1 = 0.f;
                int ol = -1;
                if (valid && !fresh) {
                    const float2 o = st[i * S + slot];
                    m0 = o.x;
                    m1 = o.y;
                    ol = lc[i * S + slot];
                }
                float nm0 = __int_as_float(0x7f800000), nm1 = nm0;
                int nloc = 0;
                unsigned npar = 0, syn = 0;
                for (int p = 0; p < dmax; p++) {
                    const bool has = p < d;
                    const int e = ra + p;
                    const int j = has ? col[e] : 0;
                    const float sv = s[j * S + slot];
                    float x = sv;
                    if (!fresh) {
                        const unsigned wb = has ? (unsigned)sg[e] : 0u;
                        const float mag = (e == ol) ? m1 : fabsf(m0);  // Obs. 1
                        const unsigned neg_eta = ((wb >> slot) & 1u) ^ (__float_as_uint(m0) >> 31);  // Obs. 2
                        x = sv - (neg_eta ? -mag : mag);  // lambda_k - eta^prev_{i,k}
                    }
                    const float ax = fabsf(x);
                    const bool lt = has && ax < nm0;  // first strict minimum (A13)
                    nm1 = lt ? nm0 : (has ? fminf(nm1, ax) : nm1);
                    nm0 = lt ? ax : nm0;
                    nloc = lt ? e : nloc;
                    const bool neg = has && x < 0.f;  // sign(0) = +1
                    npar ^= (unsigned)neg;
                    syn ^= (unsigned)(has && sv > 0.f);  // b_j = slice(s_j)
                    const unsigned bal = __ballot_sync(FULLM, neg);
                    if (has && slot == 0) sg[e] = (SWT)(S == 32 ? bal : (bal >> (sub * S)) & ((1u << S) - 1u));
                }
                if (valid) {
                    const unsigned corr = (unsigned)(d & 1) & (unsigned)(!a.literal);  // reading A1
                    st[i * S + slot] = make_float2(__uint_as_float(__float_as_uint(nm0) | ((npar ^ corr) << 31)), nm1);
                    lc[i * S + slot] = (uint16_t)nloc;
                }
                usyn |= __ballot_sync(FULLM, valid && lane_act && syn);
            }
            // fold the G sub-groups onto slot bits
            unsigned fold = 0;
#pragma unroll
            for (int q = 0; q < G; q++) fold |= (S == 32) ? usyn : ((usyn >> (q * S)) & ((1u << S) - 1u));
            if (lane == 0 && fold) atomicOr(&ctl[0], fold);
        }
        __syncthreads();

        // ---------------- D: per-slot decision, outputs of stopping slots, bit-node pass of the rest
        {
            const unsigned uns_all = ctl[0];
            unsigned fin_mask = 0, cont_mask = 0;
#pragma unroll 1
            for (int q = 0; q < S; q++) {
                if (!((active >> q) & 1u)) continue;
                const int k = slot_k[q];
                const bool uns = (uns_all >> q) & 1u;
                const bool fin = a.early ? (!uns || k == a.L) : (k == a.L);
                if (fin) fin_mask |= 1u << q;
                else cont_mask |= 1u << q;
            }
            for (unsigned fm = fin_mask; fm; fm &= fm - 1) {
                const int q = __ffs(fm) - 1;
                const int64_t f = slot_f[q];
                int be = 0;
                bool nz = false;
                for (int j = tid; j < n; j += RT) {
                    const float v = s[j * S + q];
                    const bool b = v > 0.f;  // Eq. slice
                    if (a.post) a.post[f * n + j] = v;
                    if (a.bits) a.bits[f * n + j] = (uint8_t)b;
                    be += b;
                    nz |= fabsf(v) <= 1e-4f;
                }
                for (int o = 16; o; o >>= 1) be += __shfl_xor_sync(FULLM, be, o);
                nz = __any_sync(FULLM, nz);
                if (lane == 0) {
                    if (be) atomicAdd(&slot_be[q], be);
                    if (nz) slot_nz[q] = 1;
                }
            }
            if (cont_mask) {
                const bool lane_cont = (cont_mask >> slot) & 1u;
                for (int cb = warp * G; cb < n; cb += 32 * G) {
                    const int j = cb + sub;
                    if (j >= n) continue;
                    const float rj = rs[(size_t)j * S + slot];
                    const int c0 = cp[j], dv = (int)cp[j + 1] - c0;
                    float acc = 0.f;
                    for (int q = 0; q < dv; q++) {
                        const uint32_t rc = rec[c0 + q];
                        const int e = (int)(rc >> 16), i = (int)(rc & 0xffffu);
                        const float2 o = st[i * S + slot];
                        const int ol = lc[i * S + slot];
                        const unsigned wb = (unsigned)sg[e];
                        const float mag = (e == ol) ? o.y : fabsf(o.x);
                        const unsigned neg = ((wb >> slot) & 1u) ^ (__float_as_uint(o.x) >> 31);
                        acc = acc + (neg ? -mag : mag);  // ascending rows from +0.0 (A14)
                    }
                    if (lane_cont) s[j * S + slot] = acc + rj;
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

template <int S>
void launch_s(const ResArgs &args, int ctas, size_t smem, cudaStream_t st) {
    cudaFuncSetAttribute(k_resident<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_resident<S><<<ctas, RT, smem, st>>>(args);
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
            rp.threads = RT;
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
        case 32: launch_s<32>(a, rp.ctas, rp.smem, st); break;
        case 16: launch_s<16>(a, rp.ctas, rp.smem, st); break;
        case 8: launch_s<8>(a, rp.ctas, rp.smem, st); break;
        default: launch_s<4>(a, rp.ctas, rp.smem, st); break;
    }
    return 1;
}

size_t resident_scratch_bytes(const HostGraph &g, const ResidentPlan &rp) {
    return 256 + (size_t)rp.ctas * g.n * rp.slots * 4;
}

}  // namespace ldpc
