// ldpc_internal.cuh -- internal declarations of libldpc (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/ldpc.h"

namespace ldpc {

// Frames are processed in tiles of 128 (one warp = 32 lanes x 4 frames, float4 per lane).
constexpr int TILE = 128;
constexpr int CTA = 256;  // threads per CTA of the streaming kernels (8 warps)

// Error bits raised by the ingest kernels.
enum : int { ERRB_NOT_BINARY = 1, ERRB_ROW_DEGREE = 2, ERRB_DUPLICATE = 4, ERRB_RANGE = 8 };

// Device view of the ingested Tanner graph.
struct Graph {
    int m, n, E;
    const int *row_ptr;  // [m+1]   N_i = col_idx[row_ptr[i] .. row_ptr[i+1])
    const int *col_idx;  // [E]     ascending within a row
    const int *col_ptr;  // [n+1]   M_j = bn_edge[col_ptr[j] .. col_ptr[j+1])
    const int4 *bn_edge; // [E]     {edge id e (row-list position), row i, position p in N_i, d_i & 1}
    const int2 *bn_off;  // [E]     streaming bit node, same order: {i * rs / 32, (i * rs + REC_EDGE0 + 32 p) / 32}
                         //         (row record and edge block of the edge, in 32-byte units inside a tile)
    int wr;              // sign words per row and lane in the streaming layout: ceil(max row degree / 8)
    int dmax;            // max row degree
    int dvmax;           // max column degree
};

// Per-chunk decode state of the streaming schedule, frame-interleaved in tiles of 128 slots (T tiles
// hold the chunk's frames; the workspace has Tcap >= T tiles, the extra ones receive compacted frames):
//   r, s   [Tcap][n][128] fp32       channel values and current soft vector (Eq. sCalculation)
//   rst    [Tcap][m] row records of rs bytes: the check-node state of row i for the tile's 128 slots,
//          contiguous so that a gather of one row touches one DRAM page:
//            min0 [128] fp32   |lambda| minimum of the row; SIGN BIT = row sign parity (Obs. 2)
//            min1 [128] fp32   second minimum (Obs. 1); same sign bit as min0
//            edge blocks [ecap][32 B]: byte l of edge p = sign nibble (bit v: sign of lambda_e, slot
//                              4l+v) | isloc nibble << 4 (bit v: p == min0Location of slot 4l+v)
//   unsat  [2][Tcap][4] u32          per-slot "some check unsatisfied" bits (double-buffered by body)
//   done   [Tcap][4]    u32          per-slot "stopped" bits (padding and moved-away slots are done)
//   fid    [Tcap][128]  i32          chunk frame index held by the slot (-1: none)
//   per chunk frame f < T*128: iters, conv (k and isCodeword), fcnt = fbe | fraw | fnz (bit errors,
//   raw errors, near-zero flag)
//   compaction: csrc/ccnt [Tcap] source tiles of this body and their running counts, cmap [Tcap][128]
//   (fresh slot -> source tile << 7 | slot), ctl [8] counters, work [4] persistent-sweep item counters
constexpr int REC_EDGE0 = 1024;  // byte offset of edge block 0 in a row record
enum { WK_CN = 0, WK_BN = 1, WK_MOVE = 2, WK_SYN = 3 };
enum { CT_TNEXT = 0, CT_NSRC = 1, CT_NDST = 2, CT_DBASE = 3 };
// launches of one graph-driven loop body: check node, bit node, compaction plan + move, loop step
constexpr int BODY_LAUNCHES = 5;

struct StreamState {
    int T, Tcap;
    float *r, *s;
    unsigned char *rst;  // row records
    int rs;              // bytes per row record: 1024 + 32 ecap
    uint32_t *unsat, *done;
    int *fid;
    int *iters, *conv;
    int *fcnt, *fbe, *fraw, *fnz;
    int *tcount;  // [2]     number of tiles with a running frame, per body parity
    int *tlist;   // [2][Tcap]  those tiles
    int *kdev;    // body index of the graph-driven loop
    int *work;    // [4]
    int *ctl;     // [8]
    int *csrc, *ccnt, *cmap;
    unsigned long long *nlaunch;  // [8] handle counters: [0] graph-loop launches, [1] frames moved by
                                  // compaction, [2] compactions, [3] tiles retired by them, [4] / [5]
                                  // tile-bodies swept by the check / bit node; or null
};

// ---- ingest (ingest.cu) ----
int ingest_dense(const uint8_t *H, int m, int n, cudaStream_t st, struct HostGraph *hg);
int ingest_coo(const int32_t *rows, const int32_t *cols, int64_t nnz, int m, int n, cudaStream_t st,
               struct HostGraph *hg);

struct HostGraph {  // device allocations owned by the plan
    int m = 0, n = 0, E = 0, max_row_deg = 0, max_col_deg = 0;
    int *row_ptr = nullptr, *col_idx = nullptr, *col_ptr = nullptr, *col_edge = nullptr;
    int4 *bn_edge = nullptr;
    int2 *bn_off = nullptr;  // filled at prepare once the row-record size is known (launch_bn_offsets)
    int64_t launches = 0;
    Graph view() const {
        return Graph{m, n, E, row_ptr, col_idx, col_ptr, bn_edge, bn_off, (max_row_deg + 7) / 8, max_row_deg, max_col_deg};
    }
    void free_all();
};

// ---- streaming schedule (decode_stream.cu) ----
struct StreamLaunch {
    int sms = 148;          // persistent sweep grids are multiples of the SM count
    bool cn_generic = false;  // force the any-degree check-node kernel (tests)
    bool cn_bulk = false;     // check node with cp.async.bulk row staging (rows of degree <= 32)
    size_t smem_per_sm = 0;   // shared memory per SM (bytes), for the bulk kernel's grid
    bool compact = true;    // f1: compaction of tiles with fewer than half of their frames running
    int check_every = 1;    // codeword test after body k when k % T == 0 (and after body L)
};
// edge blocks per row record for a maximum row degree (the check-node instance reads CH of them)
int edge_capacity(int dmax, bool generic);
// Launch helpers; each returns the number of kernels launched.
// the streaming bit node's per-edge record offsets for row records of rs bytes (rs % 32 == 0)
int launch_bn_offsets(const Graph &g, int rs, int2 *out, cudaStream_t st);
int launch_stage_in(const Graph &g, const StreamState &w, const float *llr, int64_t frames, cudaStream_t st);
int launch_check_node(const Graph &g, const StreamState &w, int k, bool first, bool early, bool literal,
                      const StreamLaunch &cfg, cudaStream_t st, const int *kdev = nullptr);
int launch_bit_node(const Graph &g, const StreamState &w, int k, int L, bool early, const StreamLaunch &cfg,
                    cudaStream_t st, const int *kdev = nullptr);
int launch_compact(const Graph &g, const StreamState &w, int k, const StreamLaunch &cfg, cudaStream_t st,
                   const int *kdev = nullptr);
int launch_loop_pre(const StreamState &w, int L, cudaGraphConditionalHandle h, cudaStream_t st);
int launch_loop_step(const StreamState &w, int L, cudaGraphConditionalHandle h, cudaStream_t st);
int launch_syndrome(const Graph &g, const StreamState &w, int slot, const float *sfin, const StreamLaunch &cfg,
                    cudaStream_t st);
int launch_finalize(const Graph &g, const StreamState &w, int L, int final_slot, const float *sfin, float *posterior,
                    uint8_t *bits, cudaStream_t st);
int launch_frame_stats(const StreamState &w, int64_t frames, int32_t *iters_out, uint8_t *conv_out,
                       unsigned long long *stats, cudaStream_t st);

// ---- resident schedule (decode_resident.cu) ----
struct ResidentPlan {
    bool ok = false;
    int slots = 0;       // frame slots per CTA
    int threads = 0;     // threads per CTA
    size_t smem = 0;     // dynamic shared memory bytes
    int ctas = 0;        // persistent grid size
    int dm = 0;          // max row degree (ballot-word rows)
    int dv = 0;          // max column degree
    bool regular = false;  // every row has degree dm and every column degree dv
    bool compact = false;  // compact bit-node records (larger codes, see layout_for)
    bool global_graph = false;  // Tanner-graph lists read from global memory (state only in shared memory)
};
ResidentPlan plan_resident(const HostGraph &g, bool loc16, int device);
size_t resident_scratch_bytes(const HostGraph &g, const ResidentPlan &rp);  // work counter + r scratch
int launch_resident(const Graph &g, const ResidentPlan &rp, const float *llr, int64_t frames, int L, int T, bool early,
                    bool literal, bool loc16, float *posterior, uint8_t *bits, int32_t *iters_out,
                    uint8_t *conv_out, unsigned long long *stats, int *work_counter, cudaStream_t st);

}  // namespace ldpc
