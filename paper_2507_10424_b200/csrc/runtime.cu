// runtime.cu -- host runtime behind the C-ABI of include/ldpc.h: handle, workspace, schedule choice,
// the stream-ordered loop over chunks and loop bodies, the host-buffer pipeline and kernel accounting.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "ldpc_internal.cuh"

// buffer sets of the ldpc_decode_host pipeline (LDPC_HOST_NBUF overrides the default, 2..NHB_MAX)
constexpr int NHB_MAX = 4;
constexpr int NHB_DEFAULT = 3;

using namespace ldpc;

struct ldpc_plan {
    HostGraph g;
    uint32_t flags = 0;
    int check_every = 1;
    int device = 0;
    bool poisoned = false;
    // streaming workspace
    void *ws = nullptr;
    size_t ws_bytes = 0;
    int ws_tiles = 0;
    int64_t chunk_cap = 0;  // frames per chunk, 0 = automatic
    StreamLaunch cfg;
    // resident schedule
    ResidentPlan rp;
    int *work_counter = nullptr;
    // accounting
    int64_t launches = 0;
    bool prof = false;
    struct Ev {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<Ev> evs;
    std::vector<cudaEvent_t> pool;
    int64_t prof_launches[LDPC_K_NUM_CLASSES] = {};
    double prof_ms[LDPC_K_NUM_CLASSES] = {};
    // graph-driven decode loops (one instantiated graph per distinct chunk launch)
    struct GraphEntry {
        const void *key[8];
        int64_t fc;
        int L;
        int T;
        uint32_t flags;
        void *ws;
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        uint64_t used;
    };
    std::vector<GraphEntry> graphs;
    uint64_t graph_clock = 0;
    bool use_graphs = true;
    cudaStream_t cap[2] = {nullptr, nullptr};
    // host pipeline
    cudaStream_t hs[3] = {nullptr, nullptr, nullptr};
    // ldpc_decode_host buffer sets (LLRs in, outputs back): with NHB sets the host -> device copies run up
    // to NHB - 1 chunks ahead of the decode, so a copy never waits for the copy-back of the chunk before
    void *hbuf[NHB_MAX] = {};
    size_t hbuf_bytes = 0;
    unsigned long long *hstats = nullptr;  // device counters of ldpc_decode_host (64 B, allocated once)
    // device-side accounting of graph-driven loop bodies (3 launches per body that ran)
    unsigned long long *dev_launches = nullptr;
    // completion of the handle's last enqueued work (ldpc_destroy waits for it, not for the device)
    cudaEvent_t last = nullptr;
    bool last_recorded = false;
};

namespace {

int status_of(cudaError_t e) {
    if (e == cudaSuccess) return LDPC_OK;
    if (e == cudaErrorMemoryAllocation) return LDPC_ERR_OOM;
    return LDPC_ERR_CUDA;
}

cudaEvent_t get_event(ldpc_plan *h) {
    if (!h->pool.empty()) {
        cudaEvent_t e = h->pool.back();
        h->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Launch one kernel (or a fixed group) of class `cls`, bracketed by events when profiling.
template <typename F>
void launch(ldpc_plan *h, int cls, cudaStream_t st, F &&fn) {
    if (h->prof) {
        cudaEvent_t a = get_event(h), b = get_event(h);
        cudaEventRecord(a, st);
        int nl = fn();
        cudaEventRecord(b, st);
        h->evs.push_back({cls, a, b});
        h->launches += nl;
        h->prof_launches[cls] += nl;
    } else {
        h->launches += fn();
    }
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// bytes of one row record of the streaming schedule: min0, min1 (128 fp32 each) and one 32-byte edge
// block per edge position the check-node instance reads
int row_record_bytes(const ldpc_plan *h) {
    return REC_EDGE0 + 32 * edge_capacity(h->g.max_row_deg, h->cfg.cn_generic);
}

// workspace tiles for a chunk of T tiles: room for the fresh tiles of the compactions (each one retires
// more tiles than it creates; the plan kernel never exceeds the capacity)
int tile_capacity(const ldpc_plan *h, int T) { return h->cfg.compact ? 2 * T : T; }

// Carve the workspace into its arrays (base == nullptr: only the size).  Per tile: r, s, row records,
// flags, slot frame indices, compaction map; per chunk frame: k, isCodeword, three counters.
StreamState carve(void *base, int T, int Tcap, const ldpc_plan *h, size_t *total) {
    const size_t m = h->g.m, n = h->g.n;
    char *p0 = static_cast<char *>(base);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *q = p0 ? p0 + off : nullptr;
        off += align256(bytes);
        return q;
    };

    StreamState w{};
    w.T = T;
    w.Tcap = Tcap;
    w.rs = row_record_bytes(h);
    w.r = reinterpret_cast<float *>(take((size_t)Tcap * n * TILE * 4));
    w.s = reinterpret_cast<float *>(take((size_t)Tcap * n * TILE * 4));
    w.rst = reinterpret_cast<unsigned char *>(take((size_t)Tcap * m * w.rs));
    w.unsat = reinterpret_cast<uint32_t *>(take((size_t)2 * Tcap * 16));
    w.done = reinterpret_cast<uint32_t *>(take((size_t)Tcap * 16));
    w.fid = reinterpret_cast<int *>(take((size_t)Tcap * TILE * 4));
    w.iters = reinterpret_cast<int *>(take((size_t)T * TILE * 4));
    w.conv = reinterpret_cast<int *>(take((size_t)T * TILE * 4));
    w.fcnt = reinterpret_cast<int *>(take((size_t)3 * T * TILE * 4));
    w.fbe = w.fcnt ? w.fcnt : nullptr;
    w.fraw = w.fcnt ? w.fcnt + (size_t)T * TILE : nullptr;
    w.fnz = w.fcnt ? w.fcnt + (size_t)2 * T * TILE : nullptr;
    w.tcount = reinterpret_cast<int *>(take(2 * 4));
    w.tlist = reinterpret_cast<int *>(take((size_t)2 * Tcap * 4));
    w.kdev = reinterpret_cast<int *>(take(4));
    w.work = reinterpret_cast<int *>(take(4 * 4));
    w.ctl = reinterpret_cast<int *>(take(8 * 4));
    w.csrc = reinterpret_cast<int *>(take((size_t)Tcap * 4));
    w.ccnt = reinterpret_cast<int *>(take((size_t)Tcap * 4));
    w.cmap = reinterpret_cast<int *>(take((size_t)Tcap * TILE * 4));
    w.nlaunch = h->dev_launches;
    if (total) *total = off;
    return w;
}

size_t ws_bytes_for(const ldpc_plan *h, int T) {
    size_t total = 0;
    carve(nullptr, T, tile_capacity(h, T), h, &total);
    return total;
}

int64_t auto_chunk_tiles(ldpc_plan *h) {
    size_t freeb = 0, total = 0;
    cudaMemGetInfo(&freeb, &total);
    const size_t budget = std::min<size_t>(freeb / 2 + h->ws_bytes / 2, (size_t)64 << 30);
    const size_t per = std::max<size_t>(1, ws_bytes_for(h, 1024) / 1024);  // bytes per chunk tile
    const int64_t tiles = (int64_t)(budget / per);
    return std::max<int64_t>(1, std::min<int64_t>(tiles, 32767));
}

int ensure_ws(ldpc_plan *h, int T) {
    const size_t need = ws_bytes_for(h, T);
    if (need <= h->ws_bytes) return LDPC_OK;
    for (auto &ge : h->graphs) {  // graphs embed workspace pointers
        cudaGraphExecDestroy(ge.exec);
        cudaGraphDestroy(ge.graph);
    }
    h->graphs.clear();
    if (h->ws) cudaFree(h->ws);
    h->ws = nullptr;
    h->ws_bytes = 0;
    cudaError_t e = cudaMalloc(&h->ws, need);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return LDPC_ERR_OOM;
    }
    h->ws_bytes = need;
    return LDPC_OK;
}

int check_async(ldpc_plan *h) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        h->poisoned = true;
        return LDPC_ERR_CUDA;
    }
    return LDPC_OK;
}

// kernels of a chunk graph outside the WHILE node: stage-in, body 1 (check node, bit node, compaction
// plan + move), loop_pre, final syndrome, finalize, frame stats.  Each WHILE iteration adds
// BODY_LAUNCHES (counted by the loop kernels on the device).
constexpr int GRAPH_STATIC_LAUNCHES = 9;

// One chunk as a CUDA graph: stage-in, body 1, then a conditional WHILE node whose body (check node,
// bit node, compaction, loop step) repeats while a frame is still running and k <= L, then the final
// syndrome pass and stage-out.  No host round trip and no launch for bodies after the last frame
// stopped.
template <typename Tail>
int run_graph(ldpc_plan *h, const Graph &g, const StreamState &w, const float *llr, int64_t fc, int L, bool early,
              bool literal, float *post, uint8_t *bits, int32_t *iters, uint8_t *conv, int64_t *stats,
              cudaStream_t st, Tail &&tail) {
    const void *key[8] = {llr, post, bits, iters, conv, stats, w.r, nullptr};
    for (auto &ge : h->graphs) {
        if (std::equal(key, key + 8, ge.key) && ge.fc == fc && ge.L == L && ge.flags == h->flags && ge.ws == h->ws &&
            ge.T == h->check_every) {
            ge.used = ++h->graph_clock;
            if (cudaGraphLaunch(ge.exec, st) != cudaSuccess) {
                h->poisoned = true;
                return LDPC_ERR_CUDA;
            }
            h->launches += GRAPH_STATIC_LAUNCHES;  // the loop bodies are counted on the device
            return LDPC_OK;
        }
    }
    if (!h->cap[0]) {
        for (int q = 0; q < 2; q++)
            if (cudaStreamCreateWithFlags(&h->cap[q], cudaStreamNonBlocking) != cudaSuccess) return LDPC_ERR_CUDA;
    }
    cudaStream_t c0 = h->cap[0], c1 = h->cap[1];
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(c0, cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) return status_of(e);
    launch_stage_in(g, w, llr, fc, c0);
    launch_check_node(g, w, 1, true, early, literal, h->cfg, c0);
    launch_bit_node(g, w, 1, L, early, h->cfg, c0);
    launch_compact(g, w, 1, h->cfg, c0);
    cudaStreamCaptureStatus cs;
    cudaGraph_t capg = nullptr;
    const cudaGraphNode_t *deps = nullptr;
    size_t ndeps = 0;
    e = cudaStreamGetCaptureInfo(c0, &cs, nullptr, &capg, &deps, &ndeps);
    cudaGraphConditionalHandle handle{};
    if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&handle, capg, 0, cudaGraphCondAssignDefault);
    if (e == cudaSuccess) launch_loop_pre(w, L, handle, c0);
    if (e == cudaSuccess) e = cudaStreamGetCaptureInfo(c0, &cs, nullptr, &capg, &deps, &ndeps);
    cudaGraphNode_t cond = nullptr;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    if (e == cudaSuccess) e = cudaGraphAddNode(&cond, capg, deps, ndeps, &cp);
    if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(c0, &cond, 1, cudaStreamSetCaptureDependencies);
    if (e == cudaSuccess) {
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        e = cudaStreamBeginCaptureToGraph(c1, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
        if (e == cudaSuccess) {
            launch_check_node(g, w, 2, false, early, literal, h->cfg, c1, w.kdev);
            launch_bit_node(g, w, 2, L, early, h->cfg, c1, w.kdev);
            launch_compact(g, w, 2, h->cfg, c1, w.kdev);
            launch_loop_step(w, L, handle, c1);
            cudaGraph_t out = nullptr;
            e = cudaStreamEndCapture(c1, &out);
        }
    }
    if (e == cudaSuccess) tail(c0);
    cudaError_t e2 = cudaStreamEndCapture(c0, &graph);
    if (e == cudaSuccess) e = e2;
    cudaGraphExec_t exec = nullptr;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (graph) cudaGraphDestroy(graph);
        h->use_graphs = false;  // fall back to plain stream-ordered launches on this handle
        return LDPC_ERR_UNSUPPORTED;
    }
    if (h->graphs.size() >= 32) {  // evict the least recently used graph
        size_t v = 0;
        for (size_t q = 1; q < h->graphs.size(); q++)
            if (h->graphs[q].used < h->graphs[v].used) v = q;
        cudaGraphExecDestroy(h->graphs[v].exec);
        cudaGraphDestroy(h->graphs[v].graph);
        h->graphs.erase(h->graphs.begin() + v);
    }
    ldpc_plan::GraphEntry ge;
    std::copy(key, key + 8, ge.key);
    ge.fc = fc;
    ge.L = L;
    ge.T = h->check_every;
    ge.flags = h->flags;
    ge.ws = h->ws;
    ge.graph = graph;
    ge.exec = exec;
    ge.used = ++h->graph_clock;
    h->graphs.push_back(ge);
    if (cudaGraphLaunch(exec, st) != cudaSuccess) {
        h->poisoned = true;
        return LDPC_ERR_CUDA;
    }
    h->launches += GRAPH_STATIC_LAUNCHES;
    return LDPC_OK;
}

int decode_stream(ldpc_plan *h, const float *llr, int64_t frames, int L, uint8_t *bits, int32_t *iters, float *post,
                  uint8_t *conv, int64_t *stats, cudaStream_t st) {
    const bool early = !(h->flags & LDPC_FLAG_NO_EARLY_STOP);
    const bool literal = (h->flags & LDPC_FLAG_SIGN_PAPER_LITERAL) != 0;
    const Graph g = h->g.view();
    if (!h->dev_launches) {
        if (cudaMalloc(&h->dev_launches, 8 * sizeof(unsigned long long)) != cudaSuccess) {
            cudaGetLastError();
            return LDPC_ERR_OOM;
        }
        if (cudaMemsetAsync(h->dev_launches, 0, 8 * sizeof(unsigned long long), st) != cudaSuccess)
            return LDPC_ERR_CUDA;
    }
    int64_t cap_tiles = h->chunk_cap > 0 ? (h->chunk_cap + TILE - 1) / TILE : auto_chunk_tiles(h);
    cap_tiles = std::min<int64_t>(cap_tiles, 32767);
    const int64_t need_tiles = (frames + TILE - 1) / TILE;
    const int T_max = (int)std::min<int64_t>(cap_tiles, need_tiles);
    int rc = ensure_ws(h, T_max);
    if (rc) return rc;
    const int final_slot = (L + 1) & 1;
    const bool graphs = h->use_graphs && !h->prof && L >= 2 && !(h->flags & LDPC_FLAG_NO_GRAPH);
    for (int64_t c0 = 0; c0 < frames; c0 += (int64_t)T_max * TILE) {
        const int64_t fc = std::min<int64_t>((int64_t)T_max * TILE, frames - c0);
        const int T = (int)((fc + TILE - 1) / TILE);
        const StreamState w = carve(h->ws, T, tile_capacity(h, T), h, nullptr);
        const float *sfin = L > 0 ? w.s : w.r;  // L = 0: the soft output is r itself
        const float *cl = llr + c0 * g.n;
        float *cp = post ? post + c0 * g.n : nullptr;
        uint8_t *cb = bits ? bits + c0 * g.n : nullptr;
        int32_t *ci = iters ? iters + c0 : nullptr;
        uint8_t *cc = conv ? conv + c0 : nullptr;
        auto tail = [&](cudaStream_t s2) {
            int nl = launch_syndrome(g, w, final_slot, sfin, h->cfg, s2);
            nl += launch_finalize(g, w, L, final_slot, sfin, cp, cb, s2);
            nl += launch_frame_stats(w, fc, ci, cc, reinterpret_cast<unsigned long long *>(stats), s2);
            return nl;
        };
        if (graphs && h->use_graphs) {
            rc = run_graph(h, g, w, cl, fc, L, early, literal, cp, cb, ci, cc, stats, st, tail);
            if (rc == LDPC_OK) continue;
            if (rc != LDPC_ERR_UNSUPPORTED) return rc;
        }
        launch(h, LDPC_K_STAGE_IN, st, [&] { return launch_stage_in(g, w, cl, fc, st); });
        for (int k = 1; k <= L; k++) {
            launch(h, LDPC_K_CHECK_NODE, st,
                   [&] { return launch_check_node(g, w, k, k == 1, early, literal, h->cfg, st); });
            launch(h, LDPC_K_BIT_NODE, st, [&] { return launch_bit_node(g, w, k, L, early, h->cfg, st); });
            launch(h, LDPC_K_COMPACT, st, [&] { return launch_compact(g, w, k, h->cfg, st); });
        }
        launch(h, LDPC_K_SYNDROME, st, [&] { return launch_syndrome(g, w, final_slot, sfin, h->cfg, st); });
        launch(h, LDPC_K_FINALIZE, st, [&] {
            int nl = launch_finalize(g, w, L, final_slot, sfin, cp, cb, st);
            nl += launch_frame_stats(w, fc, ci, cc, reinterpret_cast<unsigned long long *>(stats), st);
            return nl;
        });
        rc = check_async(h);
        if (rc) return rc;
    }
    return LDPC_OK;
}

bool use_resident(ldpc_plan *h) {
    if (h->flags & LDPC_FLAG_FORCE_STREAM) return false;
    if (h->flags & LDPC_FLAG_FORCE_RESIDENT) return true;
    return h->rp.ok;
}

int decode_resident(ldpc_plan *h, const float *llr, int64_t frames, int L, uint8_t *bits, int32_t *iters,
                    float *post, uint8_t *conv, int64_t *stats, cudaStream_t st) {
    if (!h->rp.ok) return LDPC_ERR_UNSUPPORTED;
    const bool early = !(h->flags & LDPC_FLAG_NO_EARLY_STOP);
    const bool literal = (h->flags & LDPC_FLAG_SIGN_PAPER_LITERAL) != 0;
    const bool loc16 = h->g.max_row_deg > 255;
    if (!h->work_counter) {
        if (cudaMalloc(&h->work_counter, resident_scratch_bytes(h->g, h->rp)) != cudaSuccess) {
            cudaGetLastError();
            return LDPC_ERR_OOM;
        }
    }
    const Graph g = h->g.view();
    // the kernel's work counter and slot frame indices are 32-bit: at most 2^30 frames per launch
    const int64_t n = g.n, cap = (int64_t)1 << 30;
    for (int64_t c0 = 0; c0 < frames; c0 += cap) {
        const int64_t fc = std::min(cap, frames - c0);
        launch(h, LDPC_K_RESIDENT, st, [&] {
            return launch_resident(g, h->rp, llr + c0 * n, fc, L, h->check_every, early, literal, loc16,
                                   post ? post + c0 * n : nullptr, bits ? bits + c0 * n : nullptr,
                                   iters ? iters + c0 : nullptr, conv ? conv + c0 : nullptr,
                                   reinterpret_cast<unsigned long long *>(stats), h->work_counter, st);
        });
    }
    return check_async(h);
}

// remember the end of the handle's last enqueued work on `st` (ldpc_destroy waits for it)
void mark_last(ldpc_plan *h, cudaStream_t st) {
    if (!h->last && cudaEventCreateWithFlags(&h->last, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        h->last = nullptr;
        return;
    }
    h->last_recorded = cudaEventRecord(h->last, st) == cudaSuccess;
}

int finish_prepare(ldpc_plan *p, int rc, uint32_t flags, ldpc_handle_t *out, cudaStream_t st) {
    if (rc != LDPC_OK) {
        p->g.free_all();
        delete p;
        return rc;
    }
    p->flags = flags;
    p->launches = p->g.launches;
    cudaGetDevice(&p->device);
    p->rp = plan_resident(p->g, p->g.max_row_deg > 255, p->device);
    cudaDeviceGetAttribute(&p->cfg.sms, cudaDevAttrMultiProcessorCount, p->device);
    if (p->cfg.sms <= 0) p->cfg.sms = 148;
    // knobs for A/B measurements and the parity tests (every variant is bit-identical)
    {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, p->device);
        p->cfg.smem_per_sm = (size_t)v;
    }
    if (const char *s = getenv("LDPC_CN_GENERIC")) p->cfg.cn_generic = atoi(s) != 0;
    if (const char *s = getenv("LDPC_CN_BULK")) p->cfg.cn_bulk = atoi(s) != 0;
    if (const char *s = getenv("LDPC_NO_COMPACT")) p->cfg.compact = atoi(s) == 0;
    if (const char *s = getenv("LDPC_NO_GRAPHS")) p->use_graphs = atoi(s) == 0;
    // the streaming bit node's edge records need the row-record size (in 32-byte units: fits int32 for any
    // workspace that fits the device)
    if (p->g.E > 0) {
        const int rs = row_record_bytes(p);
        if ((int64_t)p->g.m * (rs / 32) >= INT32_MAX ||
            cudaMalloc(&p->g.bn_off, sizeof(int2) * (size_t)p->g.E) != cudaSuccess) {
            cudaGetLastError();
            p->g.free_all();
            delete p;
            return LDPC_ERR_OOM;
        }
        p->launches += launch_bn_offsets(p->g.view(), rs, p->g.bn_off, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) {
            cudaGetLastError();
            p->g.free_all();
            delete p;
            return LDPC_ERR_CUDA;
        }
    }
    *out = p;
    return LDPC_OK;
}

}  // namespace

extern "C" {

int ldpc_abi_version(void) { return LDPC_ABI_VERSION; }

const char *ldpc_status_string(int code) {
    switch (code) {
        case LDPC_OK: return "ok";
        case LDPC_ERR_INVALID_ARG: return "invalid argument";
        case LDPC_ERR_NOT_BINARY: return "H has an entry outside {0,1}";
        case LDPC_ERR_ROW_DEGREE: return "H has a row of degree < 2";
        case LDPC_ERR_DUPLICATE_EDGE: return "H lists a (row, column) pair twice";
        case LDPC_ERR_INDEX_RANGE: return "H lists an index outside [0,m) x [0,n)";
        case LDPC_ERR_OOM: return "out of memory";
        case LDPC_ERR_CUDA: return "CUDA error (handle poisoned)";
        case LDPC_ERR_UNSUPPORTED: return "unsupported size";
        default: return "unknown status";
    }
}

int ldpc_prepare_dense(const uint8_t *H, int32_t m, int32_t n, uint32_t flags, ldpc_stream_t stream,
                       ldpc_handle_t *out) {
    if (!H || !out || m < 1 || n < 2) return LDPC_ERR_INVALID_ARG;
    ldpc_plan *p = new (std::nothrow) ldpc_plan;
    if (!p) return LDPC_ERR_OOM;
    int rc = ingest_dense(H, m, n, static_cast<cudaStream_t>(stream), &p->g);
    return finish_prepare(p, rc, flags, out, static_cast<cudaStream_t>(stream));
}

int ldpc_prepare_coo(const int32_t *rows, const int32_t *cols, int64_t nnz, int32_t m, int32_t n, uint32_t flags,
                     ldpc_stream_t stream, ldpc_handle_t *out) {
    if (!rows || !cols || !out || m < 1 || n < 2 || nnz < 0) return LDPC_ERR_INVALID_ARG;
    ldpc_plan *p = new (std::nothrow) ldpc_plan;
    if (!p) return LDPC_ERR_OOM;
    int rc = ingest_coo(rows, cols, nnz, m, n, static_cast<cudaStream_t>(stream), &p->g);
    return finish_prepare(p, rc, flags, out, static_cast<cudaStream_t>(stream));
}

int ldpc_decode(ldpc_handle_t h, const float *llr, int64_t frames, int32_t max_iter, uint8_t *bits_out,
                int32_t *iters_out, float *posterior_out, uint8_t *converged_out, int64_t *stats_inout,
                ldpc_stream_t stream) {
    if (!h || frames < 0 || max_iter < 0) return LDPC_ERR_INVALID_ARG;
    if (frames > 0 && !llr) return LDPC_ERR_INVALID_ARG;
    if (h->poisoned) return LDPC_ERR_CUDA;
    if (frames == 0) return LDPC_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int rc = use_resident(h) ? decode_resident(h, llr, frames, max_iter, bits_out, iters_out, posterior_out,
                                                     converged_out, stats_inout, st)
                                   : decode_stream(h, llr, frames, max_iter, bits_out, iters_out, posterior_out,
                                                   converged_out, stats_inout, st);
    mark_last(h, st);
    return rc;
}

int ldpc_decode_host(ldpc_handle_t h, const float *llr, int64_t frames, int32_t max_iter, uint8_t *bits_out,
                     int32_t *iters_out, float *posterior_out, uint8_t *converged_out, int64_t *stats_inout,
                     ldpc_stream_t stream) {
    if (!h || frames < 0 || max_iter < 0) return LDPC_ERR_INVALID_ARG;
    if (frames > 0 && !llr) return LDPC_ERR_INVALID_ARG;
    if (h->poisoned) return LDPC_ERR_CUDA;
    if (frames == 0) return LDPC_OK;
    const int64_t n = h->g.n;
    // chunk of frames per pipeline stage: LDPC_HOST_CHUNK_MB of LLRs (default 768 MB: enough frames per
    // decode to fill the GPU, small enough that the unoverlapped first copy and last decode + copy-back are
    // short).  Measured e2e (one B200, 55 GB/s host link; buffer sets x chunk MB): C3 2 x 384: 6.41 Gbit/s,
    // 3 x 384: 8.64, 3 x 768: 8.97 (device 9.15), 3 x 1536: 8.82, 4 x 768: 8.23; C2 2 x 384: 9.23,
    // 3 x 768: 10.91 (device 11.61)
    const char *cm = getenv("LDPC_HOST_CHUNK_MB");
    const int64_t chunk_mb = cm ? std::max(1, atoi(cm)) : 768;
    int64_t chunk = std::max<int64_t>(TILE, std::min<int64_t>(frames, (chunk_mb << 20) / (n * 4)));
    chunk = (chunk + TILE - 1) / TILE * TILE;
    const size_t per_frame = n * 4 + (bits_out ? n : 0) + (posterior_out ? n * 4 : 0) + 4 + 1;
    const size_t set_bytes = align256(chunk * n * 4) + align256(chunk * n) + align256(chunk * n * 4) +
                             align256(chunk * 4) + align256(chunk) + 256;
    (void)per_frame;
    cudaError_t e = cudaSuccess;
    if (!h->hs[0]) {
        for (int q = 0; q < 3; q++) e = cudaStreamCreateWithFlags(&h->hs[q], cudaStreamNonBlocking);
        if (e != cudaSuccess) return status_of(e);
    }
    const char *nb = getenv("LDPC_HOST_NBUF");
    const int nhb = nb ? std::min(NHB_MAX, std::max(2, atoi(nb))) : NHB_DEFAULT;
    if (h->hbuf_bytes < set_bytes || !h->hbuf[nhb - 1]) {
        for (int q = 0; q < NHB_MAX; q++) {
            cudaFree(h->hbuf[q]);
            h->hbuf[q] = nullptr;
        }
        h->hbuf_bytes = 0;
        for (int q = 0; q < nhb; q++)
            if (cudaMalloc(&h->hbuf[q], set_bytes) != cudaSuccess) {
                cudaGetLastError();
                return LDPC_ERR_OOM;
            }
        h->hbuf_bytes = set_bytes;
    }
    if (stats_inout && !h->hstats) {
        if (cudaMalloc(&h->hstats, 64) != cudaSuccess) {
            cudaGetLastError();
            h->hstats = nullptr;
            return LDPC_ERR_OOM;
        }
    }
    // every allocation is done: from here on, all paths return the events to the pool
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    cudaStream_t s_in = h->hs[0], s_run = h->hs[1], s_out = h->hs[2];
    cudaEvent_t ev_start = get_event(h), ev_in[NHB_MAX], ev_run[NHB_MAX], ev_out[NHB_MAX];
    for (int q = 0; q < nhb; q++) {
        ev_in[q] = get_event(h);
        ev_run[q] = get_event(h);
        ev_out[q] = get_event(h);
    }
    cudaEventRecord(ev_start, user);
    cudaStreamWaitEvent(s_in, ev_start, 0);
    cudaStreamWaitEvent(s_run, ev_start, 0);
    cudaStreamWaitEvent(s_out, ev_start, 0);
    unsigned long long *d_stats = stats_inout ? h->hstats : nullptr;
    if (d_stats) cudaMemsetAsync(d_stats, 0, 64, s_run);
    int rc = LDPC_OK;
    int idx = 0, last = 0;
    bool used[NHB_MAX] = {};
    // chunk sizes ramp up geometrically from chunk/16 (the first copy, which nothing overlaps, is short)
    int64_t cur = std::max<int64_t>(TILE, (chunk / 16 + TILE - 1) / TILE * TILE);
    for (int64_t c0 = 0, fc = 0; c0 < frames && rc == LDPC_OK; c0 += fc, idx = (idx + 1) % nhb, cur = std::min(chunk, 2 * cur)) {
        last = idx;
        fc = std::min(cur, frames - c0);
        char *base = static_cast<char *>(h->hbuf[idx]);
        float *d_llr = reinterpret_cast<float *>(base);
        uint8_t *d_bits = reinterpret_cast<uint8_t *>(base + align256(chunk * n * 4));
        float *d_post = reinterpret_cast<float *>(base + align256(chunk * n * 4) + align256(chunk * n));
        int32_t *d_iters = reinterpret_cast<int32_t *>(base + align256(chunk * n * 4) + align256(chunk * n) +
                                                      align256(chunk * n * 4));
        uint8_t *d_conv = reinterpret_cast<uint8_t *>(reinterpret_cast<char *>(d_iters) + align256(chunk * 4));
        if (used[idx]) cudaStreamWaitEvent(s_in, ev_out[idx], 0);  // buffer set free again
        cudaMemcpyAsync(d_llr, llr + c0 * n, fc * n * 4, cudaMemcpyHostToDevice, s_in);
        cudaEventRecord(ev_in[idx], s_in);
        cudaStreamWaitEvent(s_run, ev_in[idx], 0);
        rc = ldpc_decode(h, d_llr, fc, max_iter, bits_out ? d_bits : nullptr, iters_out ? d_iters : nullptr,
                         posterior_out ? d_post : nullptr, converged_out ? d_conv : nullptr,
                         reinterpret_cast<int64_t *>(d_stats), s_run);
        cudaEventRecord(ev_run[idx], s_run);
        cudaStreamWaitEvent(s_out, ev_run[idx], 0);
        if (bits_out) cudaMemcpyAsync(bits_out + c0 * n, d_bits, fc * n, cudaMemcpyDeviceToHost, s_out);
        if (posterior_out) cudaMemcpyAsync(posterior_out + c0 * n, d_post, fc * n * 4, cudaMemcpyDeviceToHost, s_out);
        if (iters_out) cudaMemcpyAsync(iters_out + c0, d_iters, fc * 4, cudaMemcpyDeviceToHost, s_out);
        if (converged_out) cudaMemcpyAsync(converged_out + c0, d_conv, fc, cudaMemcpyDeviceToHost, s_out);
        cudaEventRecord(ev_out[idx], s_out);
        used[idx] = true;
    }
    int64_t hstats[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (d_stats) {
        cudaStreamWaitEvent(s_out, ev_run[last], 0);
        cudaMemcpyAsync(hstats, d_stats, 64, cudaMemcpyDeviceToHost, s_out);
    }
    e = cudaStreamSynchronize(s_out);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s_run);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s_in);
    h->pool.push_back(ev_start);
    for (int q = 0; q < nhb; q++) {
        h->pool.push_back(ev_in[q]);
        h->pool.push_back(ev_run[q]);
        h->pool.push_back(ev_out[q]);
    }
    if (rc) return rc;
    if (e != cudaSuccess) {
        h->poisoned = true;
        return LDPC_ERR_CUDA;
    }
    if (stats_inout)
        for (int q = 0; q < 8; q++) stats_inout[q] += hstats[q];
    return LDPC_OK;
}

int ldpc_info(ldpc_handle_t h, int32_t *m, int32_t *n, int64_t *nnz, int32_t *max_row_deg, int32_t *max_col_deg) {
    if (!h) return LDPC_ERR_INVALID_ARG;
    if (m) *m = h->g.m;
    if (n) *n = h->g.n;
    if (nnz) *nnz = h->g.E;
    if (max_row_deg) *max_row_deg = h->g.max_row_deg;
    if (max_col_deg) *max_col_deg = h->g.max_col_deg;
    return LDPC_OK;
}

int ldpc_get_graph(ldpc_handle_t h, int32_t *row_ptr, int32_t *col_idx, int32_t *col_ptr, int32_t *col_edge) {
    if (!h) return LDPC_ERR_INVALID_ARG;
    if (h->poisoned) return LDPC_ERR_CUDA;
    cudaError_t e = cudaSuccess;
    if (row_ptr && e == cudaSuccess) e = cudaMemcpy(row_ptr, h->g.row_ptr, sizeof(int) * (h->g.m + 1), cudaMemcpyDeviceToHost);
    if (col_idx && e == cudaSuccess) e = cudaMemcpy(col_idx, h->g.col_idx, sizeof(int) * h->g.E, cudaMemcpyDeviceToHost);
    if (col_ptr && e == cudaSuccess) e = cudaMemcpy(col_ptr, h->g.col_ptr, sizeof(int) * (h->g.n + 1), cudaMemcpyDeviceToHost);
    if (col_edge && e == cudaSuccess) e = cudaMemcpy(col_edge, h->g.col_edge, sizeof(int) * h->g.E, cudaMemcpyDeviceToHost);
    return status_of(e);
}

int ldpc_set_flags(ldpc_handle_t h, uint32_t flags) {
    if (!h) return LDPC_ERR_INVALID_ARG;
    h->flags = flags;
    return LDPC_OK;
}

int ldpc_set_check_every(ldpc_handle_t h, int32_t T) {
    if (!h || T < 1) return LDPC_ERR_INVALID_ARG;
    h->check_every = T;
    h->cfg.check_every = T;
    return LDPC_OK;
}

int ldpc_set_chunk(ldpc_handle_t h, int64_t frames_per_chunk) {
    if (!h || frames_per_chunk < 0) return LDPC_ERR_INVALID_ARG;
    h->chunk_cap = frames_per_chunk;
    return LDPC_OK;
}

int ldpc_schedule(ldpc_handle_t h) {
    if (!h) return LDPC_ERR_INVALID_ARG;
    if (!use_resident(h)) return 0;
    return h->rp.ok ? 1 : LDPC_ERR_UNSUPPORTED;
}

int ldpc_profile_enable(ldpc_handle_t h, int enable) {
    if (!h) return LDPC_ERR_INVALID_ARG;
    h->prof = enable != 0;
    return LDPC_OK;
}

int ldpc_profile_read(ldpc_handle_t h, int64_t *launches, double *ms) {
    if (!h) return LDPC_ERR_INVALID_ARG;
    for (auto &ev : h->evs) {
        cudaError_t e = cudaEventSynchronize(ev.b);
        float t = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t, ev.a, ev.b);
        if (e != cudaSuccess) {
            h->poisoned = true;
            return LDPC_ERR_CUDA;
        }
        h->prof_ms[ev.cls] += t;
        h->pool.push_back(ev.a);
        h->pool.push_back(ev.b);
    }
    h->evs.clear();
    for (int c = 0; c < LDPC_K_NUM_CLASSES; c++) {
        if (launches) launches[c] = h->prof_launches[c];
        if (ms) ms[c] = h->prof_ms[c];
    }
    return LDPC_OK;
}

int ldpc_profile_reset(ldpc_handle_t h) {
    if (!h) return LDPC_ERR_INVALID_ARG;
    int rc = ldpc_profile_read(h, nullptr, nullptr);
    for (int c = 0; c < LDPC_K_NUM_CLASSES; c++) {
        h->prof_launches[c] = 0;
        h->prof_ms[c] = 0.0;
    }
    return rc;
}

int ldpc_stream_counters(ldpc_handle_t h, int64_t *counters) {
    if (!h || !counters) return LDPC_ERR_INVALID_ARG;
    unsigned long long c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (h->dev_launches) {
        cudaError_t e = cudaDeviceSynchronize();
        if (e == cudaSuccess) e = cudaMemcpy(c, h->dev_launches, sizeof(c), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            h->poisoned = true;
            return LDPC_ERR_CUDA;
        }
    }
    for (int q = 0; q < 5; q++) counters[q] = (int64_t)c[q + 1];
    return LDPC_OK;
}

int64_t ldpc_launch_count(ldpc_handle_t h) {
    if (!h) return -1;
    unsigned long long dev = 0;
    if (h->dev_launches) {  // loop bodies launched by graph conditional nodes (synchronises the device)
        if (cudaDeviceSynchronize() != cudaSuccess ||
            cudaMemcpy(&dev, h->dev_launches, sizeof(dev), cudaMemcpyDeviceToHost) != cudaSuccess) {
            cudaGetLastError();
            dev = 0;
        }
    }
    return h->launches + (int64_t)dev;
}

void ldpc_destroy(ldpc_handle_t h) {
    if (!h) return;
    // wait for this handle's own work only (its last decode and its internal streams), not the device
    if (h->last) {
        if (h->last_recorded) cudaEventSynchronize(h->last);
        cudaEventDestroy(h->last);
    }
    for (int q = 0; q < 3; q++)
        if (h->hs[q]) cudaStreamSynchronize(h->hs[q]);
    for (int q = 0; q < 2; q++)
        if (h->cap[q]) cudaStreamSynchronize(h->cap[q]);
    h->g.free_all();
    cudaFree(h->hstats);
    cudaFree(h->dev_launches);
    cudaFree(h->ws);
    cudaFree(h->work_counter);
    for (int q = 0; q < NHB_MAX; q++) cudaFree(h->hbuf[q]);
    for (int q = 0; q < 3; q++)
        if (h->hs[q]) cudaStreamDestroy(h->hs[q]);
    for (auto &ev : h->evs) {
        cudaEventDestroy(ev.a);
        cudaEventDestroy(ev.b);
    }
    for (auto e : h->pool) cudaEventDestroy(e);
    for (auto &ge : h->graphs) {
        cudaGraphExecDestroy(ge.exec);
        cudaGraphDestroy(ge.graph);
    }
    for (int q = 0; q < 2; q++)
        if (h->cap[q]) cudaStreamDestroy(h->cap[q]);
    cudaGetLastError();
    delete h;
}

}  // extern "C"
