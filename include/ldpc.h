/*
 * ldpc.h -- C-ABI of libldpc: batched Min-Sum LDPC decoding on NVIDIA B200 (sm_100a)
 * with the parity matrix H passed as a runtime argument.
 *
 * The problem statement this library implements is Algorithm 1 / Algorithm 2 of
 * arXiv 2507.10424 (PAPER.md, "P:n" = line n):
 *   Input  "The parity matrix H, the received vector r and the maximum number of
 *           iterations L".
 *   Output "A binary vector b, the iteration number at which the decoder stopped k,
 *           a status indication isCodeword", plus the final soft vector s
 *           (Eq. sCalculation).
 * The decoder depends only on H's dimensions m x n (P:5): H is ingested at run
 * time into edge lists, no kernel is specialised on H's content.
 *
 * Conventions shared with the CPU oracle:
 *   - LLR sign: strictly positive means logical 1, non-positive means 0;
 *     slicing b_j = (s_j > 0) (Eq. slice).
 *   - Check-node update Eq. eta_update computed through Observations 1 and 2
 *     (P:183-230): min0, min0Location, min1 and the sign parity of each row, with
 *     sign(0) = +1.  Default sign rule CORRECTED multiplies by (-1)^{d_i}
 *     (reading A1); LDPC_FLAG_SIGN_PAPER_LITERAL drops that factor.
 *   - Bit-node update Eq. lambda_j: acc = +0.0f, acc += eta_{i,j} over the
 *     rows i of column j in ascending order, then s_j = acc + r_j (reading A14).
 *   - A pre-loop codeword test (Listing 1): a frame whose sliced input is a
 *     codeword stops with k = 0.  Each later loop body increments k; a frame
 *     stops as soon as H.b = 0 (mod 2), or after L bodies.
 *   - All arithmetic is IEEE fp32 (reading A14), bit-identical to the oracle.
 *
 * General rules:
 *   - Every pointer argument is a DEVICE pointer unless the comment says "host".
 *   - Every call taking an ldpc_stream_t is stream-ordered on that stream (a
 *     cudaStream_t cast to void*; NULL = the legacy default stream).
 *   - Return value: LDPC_OK (0) or a negative ldpc_status code.  Argument errors return
 *     before anything is enqueued.  An asynchronous CUDA failure is reported as
 *     LDPC_ERR_CUDA by the call that observes it and poisons the handle (every later
 *     call on it returns LDPC_ERR_CUDA; only ldpc_destroy remains valid).
 *   - Ownership: the caller owns every buffer it passes; the handle owns the ingested
 *     graph and its decode workspace and frees them in ldpc_destroy.
 *   - Thread safety: one call in flight per handle (not re-entrant); many handles may
 *     coexist, on one device or several (one per process under torch.distributed).
 */
#ifndef LDPC_H
#define LDPC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LDPC_ABI_VERSION 1

#if defined(__GNUC__)
#define LDPC_API __attribute__((visibility("default")))
#else
#define LDPC_API
#endif

typedef struct ldpc_plan *ldpc_handle_t;
typedef void *ldpc_stream_t; /* cudaStream_t */

enum ldpc_status {
    LDPC_OK = 0,
    LDPC_ERR_INVALID_ARG = -1,    /* null required pointer, m < 1, n < 2, frames < 0, max_iter < 0 */
    LDPC_ERR_NOT_BINARY = -2,     /* a dense H entry outside {0,1} */
    LDPC_ERR_ROW_DEGREE = -3,     /* a row of H with fewer than 2 ones (leave-one-out undefined) */
    LDPC_ERR_DUPLICATE_EDGE = -4, /* a repeated (i,j) in the COO list */
    LDPC_ERR_INDEX_RANGE = -5,    /* a COO index outside [0,m) x [0,n) */
    LDPC_ERR_OOM = -6,            /* device or pinned-host allocation failed */
    LDPC_ERR_CUDA = -7,           /* a CUDA runtime error; the handle is poisoned */
    LDPC_ERR_UNSUPPORTED = -8     /* size beyond the implementation limits (nnz >= 2^31, row degree > 65535) */
};

enum ldpc_flags {
    LDPC_FLAG_SIGN_PAPER_LITERAL = 1u, /* drop the (-1)^{d_i} factor of reading A1 (debug / paper-literal mode) */
    LDPC_FLAG_NO_EARLY_STOP = 2u,      /* no pre-check, no early exit: every frame runs exactly max_iter
                                          bodies; converged = (H.b == 0) after the last body */
    LDPC_FLAG_FORCE_STREAM = 4u,       /* always use the HBM-streaming schedule (per-iteration CN/BN sweeps) */
    LDPC_FLAG_FORCE_RESIDENT = 8u,     /* always use the SMEM-resident schedule (fails with UNSUPPORTED if the
                                          per-frame state of H does not fit shared memory) */
    LDPC_FLAG_NO_GRAPH = 16u           /* streaming schedule: issue every loop body as plain stream-ordered
                                          launches instead of one CUDA graph per chunk (whose conditional
                                          WHILE node stops launching bodies once every frame has stopped) */
};

/*
 * Ingest a dense 0/1 parity matrix.  H: device, m*n bytes, row-major (H[i*n + j] = H(i,j)).
 * Builds, on the device, the row lists N_i (ascending columns) and the column
 * lists M_j (ascending rows).  Synchronous on `stream` (the edge count must be
 * known to size the lists).  H may be freed when the call returns.
 * Errors: INVALID_ARG, NOT_BINARY, ROW_DEGREE, OOM, CUDA, UNSUPPORTED.  *out is set only on success.
 */
LDPC_API int ldpc_prepare_dense(const uint8_t *H, int32_t m, int32_t n, uint32_t flags, ldpc_stream_t stream,
                       ldpc_handle_t *out);

/*
 * Ingest H as the list of its ones: rows[t], cols[t] (device int32, 0-based), t < nnz, any order.
 * Same semantics and synchronisation as ldpc_prepare_dense.
 * Errors: INVALID_ARG, INDEX_RANGE, DUPLICATE_EDGE, ROW_DEGREE, OOM, CUDA, UNSUPPORTED.
 */
LDPC_API int ldpc_prepare_coo(const int32_t *rows, const int32_t *cols, int64_t nnz, int32_t m, int32_t n, uint32_t flags,
                     ldpc_stream_t stream, ldpc_handle_t *out);

/*
 * Decode `frames` independent frames (Alg. 1) with at most max_iter loop bodies.
 *   llr           [frames][n] fp32, frame-major: the received vectors r (finite values).
 *   bits_out      [frames][n] uint8 0/1: the hard decision b of the final soft vector, or NULL.
 *   iters_out     [frames] int32: k, the number of completed loop bodies (0 if the pre-check passes), or NULL.
 *   posterior_out [frames][n] fp32: the final soft vector s, or NULL.
 *   converged_out [frames] uint8: isCodeword (H.b == 0 for the returned b), or NULL.
 *   stats_inout   int64[8] ACCUMULATED (+=), or NULL: [0] frames, [1] bit errors (ones of b, the
 *                 all-zero codeword being sent), [2] frame errors (frames with a one in b),
 *                 [3] undetected errors (converged frames with a one in b), [4] sum of k,
 *                 [5] converged frames, [6] near-zero frames (min_j |s_j| <= 1e-4),
 *                 [7] raw bit errors (r_j > 0).
 * Stream-ordered, no host synchronisation; frames == 0 is a no-op.  Each frame's outputs are
 * independent of the batch it is decoded in.  Larger batches are processed in
 * chunks of the handle's workspace.
 * Errors: INVALID_ARG, OOM, CUDA.
 */
LDPC_API int ldpc_decode(ldpc_handle_t h, const float *llr, int64_t frames, int32_t max_iter, uint8_t *bits_out,
                int32_t *iters_out, float *posterior_out, uint8_t *converged_out, int64_t *stats_inout,
                ldpc_stream_t stream);

/*
 * Same as ldpc_decode, but every buffer is in HOST memory (pageable or pinned); stats_inout is host too.
 * Chunks are copied host->device, decoded and copied back with the copies of one chunk overlapping
 * the decode of another (three internal streams ordered after `stream`: copy-in, decode, copy-out; three
 * device buffer sets rotate, so the copy-in runs up to two chunks ahead of the decode and never waits for
 * a copy-back; environment LDPC_HOST_NBUF = 2..4 and LDPC_HOST_CHUNK_MB override the set count and the
 * 768 MB chunk of LLRs).  Synchronous: returns when the outputs are in host memory.
 */
LDPC_API int ldpc_decode_host(ldpc_handle_t h, const float *llr, int64_t frames, int32_t max_iter, uint8_t *bits_out,
                     int32_t *iters_out, float *posterior_out, uint8_t *converged_out, int64_t *stats_inout,
                     ldpc_stream_t stream);

/* Dimensions and degree extremes of the ingested H (host outputs; any may be NULL). */
LDPC_API int ldpc_info(ldpc_handle_t h, int32_t *m, int32_t *n, int64_t *nnz, int32_t *max_row_deg, int32_t *max_col_deg);

/*
 * Copy the ingested adjacency to HOST arrays (for verification): row_ptr[m+1], col_idx[nnz]
 * (N_i ascending), col_ptr[n+1], col_edge[nnz] (for each column, the row-list positions of its
 * ones in ascending row order).  Any pointer may be NULL.  Synchronous.
 */
LDPC_API int ldpc_get_graph(ldpc_handle_t h, int32_t *row_ptr, int32_t *col_idx, int32_t *col_ptr, int32_t *col_edge);

/* Replace the handle's flags (ldpc_flags) for later decodes. */
LDPC_API int ldpc_set_flags(ldpc_handle_t h, uint32_t flags);

/*
 * Codeword-test interval T >= 1 for later decodes (default 1 = Alg. 1): the test after loop
 * body k runs when k % T == 0 or k == max_iter; the pre-loop test (k = 0) always runs.  T = 6 is the
 * paper's experimental setting ("Termination was checked for every 6 iterations").
 * Errors: INVALID_ARG (T < 1).
 */
LDPC_API int ldpc_set_check_every(ldpc_handle_t h, int32_t T);

/* Cap the frames processed per workspace chunk (0 = automatic).  Rounded up to a multiple of 128. */
LDPC_API int ldpc_set_chunk(ldpc_handle_t h, int64_t frames_per_chunk);

/* Which schedule ldpc_decode uses for this handle: 0 = HBM streaming, 1 = SMEM resident,
 * LDPC_ERR_UNSUPPORTED if LDPC_FLAG_FORCE_RESIDENT is set but H's per-frame state does not fit SMEM. */
LDPC_API int ldpc_schedule(ldpc_handle_t h);

/*
 * Kernel accounting.  With profiling enabled, every kernel launch of ldpc_decode is bracketed by
 * CUDA events on the launching stream; ldpc_profile_read synchronises and returns, per kernel class
 * (see ldpc_kernel_class), the launch count and the summed device milliseconds since the last reset.
 * The launch counter counts every kernel launched by the handle whether profiling is on or not.
 */
enum ldpc_kernel_class {
    LDPC_K_INGEST = 0,
    LDPC_K_STAGE_IN = 1,
    LDPC_K_CHECK_NODE = 2,
    LDPC_K_BIT_NODE = 3,
    LDPC_K_SYNDROME = 4,
    LDPC_K_FINALIZE = 5,
    LDPC_K_RESIDENT = 6,
    LDPC_K_COMPACT = 7, /* streaming schedule: compaction of tiles with few running frames (plan + move) */
    LDPC_K_NUM_CLASSES = 8
};
LDPC_API int ldpc_profile_enable(ldpc_handle_t h, int enable);
LDPC_API int ldpc_profile_read(ldpc_handle_t h, int64_t *launches /* [LDPC_K_NUM_CLASSES] */,
                      double *milliseconds /* [LDPC_K_NUM_CLASSES] */);
LDPC_API int ldpc_profile_reset(ldpc_handle_t h);
/* Kernels launched by the handle so far, including the loop bodies a CUDA-graph conditional node ran
 * (counted on the device: this call synchronises the device). */
LDPC_API int64_t ldpc_launch_count(ldpc_handle_t h);

/*
 * Work counters of the streaming schedule since the handle was created (tiles with fewer
 * than half of their frames running have those frames moved into fresh dense tiles): counters[0] frames
 * moved, [1] compactions, [2] source tiles retired, [3] tile-bodies swept by the check node (tiles of 128
 * slots x loop bodies), [4] tile-bodies swept by the bit node.  Host output; synchronises the device.
 * Errors: INVALID_ARG, CUDA.
 */
LDPC_API int ldpc_stream_counters(ldpc_handle_t h, int64_t *counters /* [5] */);

LDPC_API void ldpc_destroy(ldpc_handle_t h);
LDPC_API const char *ldpc_status_string(int code);
LDPC_API int ldpc_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LDPC_H */
