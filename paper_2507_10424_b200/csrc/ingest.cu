// ingest.cu -- step a1: build the Tanner graph of a runtime H on the device.
//
// N_i = {b_j : H(i,j) = 1} becomes a row CSR with ascending columns; M_j = {c_i : H(i,j) = 1}
// becomes, per column, the list of its edges in ascending row order, each carrying the
// edge id (row-list position), the row, the position inside N_i and the parity of d_i -- everything
// the bit-node sweep needs to rebuild eta_{i,j} from the compressed row state.  Nothing is
// specialised on H's content (P:5): only m, n and the list of ones drive the kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "ldpc_internal.cuh"

namespace ldpc {

namespace {

__global__ void k_dense_count(const uint8_t *__restrict__ H, int m, int n, int *__restrict__ row_deg,
                              int *__restrict__ err, unsigned long long *__restrict__ total) {
    // one warp per row; lanes stride the columns (coalesced byte loads)
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= m) return;
    const uint8_t *row = H + (size_t)warp * n;
    int cnt = 0, bad = 0;
    for (int j = lane; j < n; j += 32) {
        uint8_t v = __ldg(row + j);
        cnt += (v != 0);
        bad |= (v > 1);
    }
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if (lane == 0) {
        row_deg[warp] = cnt;
        if (cnt) atomicAdd(total, (unsigned long long)cnt);  // E in 64 bits (a dense H may exceed 2^31 ones)
        if (bad) atomicOr(err, ERRB_NOT_BINARY);
    }
}

__global__ void k_dense_fill(const uint8_t *__restrict__ H, int m, int n, const int *__restrict__ row_ptr,
                             int *__restrict__ col_idx) {
    // ballot compaction keeps the columns of each row in ascending order
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= m) return;
    const uint8_t *row = H + (size_t)warp * n;
    int base = row_ptr[warp];
    for (int j0 = 0; j0 < n; j0 += 32) {
        int j = j0 + lane;
        bool one = j < n && __ldg(row + j) != 0;
        unsigned mask = __ballot_sync(0xffffffffu, one);
        if (one) col_idx[base + __popc(mask & ((1u << lane) - 1u))] = j;
        base += __popc(mask);
    }
}

__global__ void k_coo_count(const int32_t *__restrict__ rows, const int32_t *__restrict__ cols, int64_t nnz, int m,
                            int n, int *__restrict__ row_deg, int *__restrict__ err) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nnz) return;
    int i = rows[t], j = cols[t];
    if (i < 0 || i >= m || j < 0 || j >= n) {
        atomicOr(err, ERRB_RANGE);
        return;
    }
    atomicAdd(row_deg + i, 1);
}

__global__ void k_coo_fill(const int32_t *__restrict__ rows, const int32_t *__restrict__ cols, int64_t nnz,
                           const int *__restrict__ row_ptr, int *__restrict__ cursor, int *__restrict__ col_idx) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nnz) return;
    int i = rows[t];
    int slot = atomicAdd(cursor + i, 1);
    col_idx[row_ptr[i] + slot] = cols[t];
}

// after the segmented sort: equal neighbours inside a segment are duplicates; longest segment
__global__ void k_seg_check(const int *__restrict__ ptr, int count, const int *__restrict__ vals,
                            int *__restrict__ err, int *__restrict__ max_len) {
    const int sgm = blockIdx.x * blockDim.x + threadIdx.x;
    if (sgm >= count) return;
    const int a = ptr[sgm], b = ptr[sgm + 1];
    for (int x = a + 1; x < b; x++)
        if (vals[x] == vals[x - 1]) {
            atomicOr(err, ERRB_DUPLICATE);
            break;
        }
    atomicMax(max_len, b - a);
}

// per row: degree check, max row degree, column degree counts, edge -> (row, position, parity)
__global__ void k_rows_finish(const int *__restrict__ row_ptr, const int *__restrict__ col_idx, int m,
                              int *__restrict__ col_deg, int *__restrict__ edge_row, int *__restrict__ edge_pos,
                              int *__restrict__ err, int *__restrict__ max_row) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    int a = row_ptr[i], b = row_ptr[i + 1];
    if (b - a < 2) atomicOr(err, ERRB_ROW_DEGREE);
    atomicMax(max_row, b - a);
    for (int e = a; e < b; e++) {
        atomicAdd(col_deg + col_idx[e], 1);
        edge_row[e] = i;
        edge_pos[e] = e - a;
    }
}

__global__ void k_col_fill(const int *__restrict__ col_idx, int E, const int *__restrict__ col_ptr,
                           int *__restrict__ cursor, int *__restrict__ col_edge) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    int j = col_idx[e];
    int slot = atomicAdd(cursor + j, 1);
    col_edge[col_ptr[j] + slot] = e;
}

__global__ void k_bn_edges(const int *__restrict__ col_edge, int E, const int *__restrict__ edge_row,
                           const int *__restrict__ edge_pos, const int *__restrict__ row_ptr, int4 *__restrict__ out) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= E) return;
    int e = col_edge[q];
    int i = edge_row[e];
    int d = row_ptr[i + 1] - row_ptr[i];
    out[q] = make_int4(e, i, edge_pos[e], d & 1);
}

int cuda_status(cudaError_t e) {
    if (e == cudaErrorMemoryAllocation) return LDPC_ERR_OOM;
    return e == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

#define CK(x)                                  \
    do {                                       \
        cudaError_t _e = (x);                  \
        if (_e != cudaSuccess) {               \
            on_error();                        \
            return cuda_status(_e);            \
        }                                      \
    } while (0)

int blocks(int64_t work, int per) { return (int)std::max<int64_t>(1, (work + per - 1) / per); }

// Common tail: from a filled row CSR build the column lists and the BN edge records.
struct Builder {
    HostGraph *hg;
    cudaStream_t st;
    int *row_deg = nullptr, *err = nullptr, *maxes = nullptr, *col_deg = nullptr, *cursor = nullptr,
        *edge_row = nullptr, *edge_pos = nullptr, *keys_tmp = nullptr;
    void *temp = nullptr;  // CUB scratch
    size_t temp_bytes = 0;
    void scratch_free() {
        cudaFree(row_deg); cudaFree(err); cudaFree(maxes); cudaFree(col_deg); cudaFree(cursor);
        cudaFree(edge_row); cudaFree(edge_pos); cudaFree(keys_tmp); cudaFree(temp);
        row_deg = err = maxes = col_deg = cursor = edge_row = edge_pos = keys_tmp = nullptr;
        temp = nullptr;
        temp_bytes = 0;
    }
    int need_temp(size_t bytes) {
        if (bytes <= temp_bytes) return LDPC_OK;
        cudaFree(temp);
        temp = nullptr;
        temp_bytes = 0;
        CK(cudaMalloc(&temp, std::max<size_t>(bytes, 256)));
        temp_bytes = std::max<size_t>(bytes, 256);
        return LDPC_OK;
    }
    // out[0] = 0, out[k+1] = in[0] + ... + in[k]: a device-wide scan (any count)
    int scan(const int *in, int count, int *out) {
        CK(cudaMemsetAsync(out, 0, sizeof(int), st));
        if (count == 0) return LDPC_OK;
        size_t bytes = 0;
        CK(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out + 1, count, st));
        if (int rc = need_temp(bytes)) return rc;
        CK(cub::DeviceScan::InclusiveSum(temp, bytes, in, out + 1, count, st));
        hg->launches += 2;
        return LDPC_OK;
    }
    // sort every segment [ptr[q], ptr[q+1]) of vals ascending (a segmented sort: any segment length), then
    // flag repeated values and record the longest segment in *max_len
    int sort_segments(int *vals, int E, const int *ptr, int count, int *max_len) {
        if (E > 1) {
            if (!keys_tmp) CK(cudaMalloc(&keys_tmp, sizeof(int) * (size_t)E));
            size_t bytes = 0;
            CK(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, vals, keys_tmp, E, count, ptr, ptr + 1, st));
            if (int rc = need_temp(bytes)) return rc;
            CK(cub::DeviceSegmentedSort::SortKeys(temp, bytes, vals, keys_tmp, E, count, ptr, ptr + 1, st));
            CK(cudaMemcpyAsync(vals, keys_tmp, sizeof(int) * (size_t)E, cudaMemcpyDeviceToDevice, st));
            hg->launches += 3;
        }
        k_seg_check<<<blocks(count, 256), 256, 0, st>>>(ptr, count, vals, err, max_len);
        hg->launches += 1;
        CK(cudaGetLastError());
        return LDPC_OK;
    }
    void on_error() {
        scratch_free();
        hg->free_all();
    }
    int fail(int code) {
        on_error();
        return code;
    }
    int read_err() {
        int h_err = 0;
        cudaError_t e = cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail(cuda_status(e));
        if (h_err & ERRB_NOT_BINARY) return fail(LDPC_ERR_NOT_BINARY);
        if (h_err & ERRB_RANGE) return fail(LDPC_ERR_INDEX_RANGE);
        if (h_err & ERRB_DUPLICATE) return fail(LDPC_ERR_DUPLICATE_EDGE);
        if (h_err & ERRB_ROW_DEGREE) return fail(LDPC_ERR_ROW_DEGREE);
        return LDPC_OK;
    }
    int columns() {
        const int m = hg->m, n = hg->n, E = hg->E;
        CK(cudaMalloc(&col_deg, sizeof(int) * n));
        CK(cudaMalloc(&cursor, sizeof(int) * std::max(m, n)));
        CK(cudaMalloc(&edge_row, sizeof(int) * std::max(E, 1)));
        CK(cudaMalloc(&edge_pos, sizeof(int) * std::max(E, 1)));
        CK(cudaMalloc(&hg->col_ptr, sizeof(int) * (n + 1)));
        CK(cudaMalloc(&hg->col_edge, sizeof(int) * std::max(E, 1)));
        CK(cudaMalloc(&hg->bn_edge, sizeof(int4) * std::max(E, 1)));
        CK(cudaMemsetAsync(col_deg, 0, sizeof(int) * n, st));
        CK(cudaMemsetAsync(cursor, 0, sizeof(int) * std::max(m, n), st));
        k_rows_finish<<<blocks(m, 256), 256, 0, st>>>(hg->row_ptr, hg->col_idx, m, col_deg, edge_row, edge_pos, err,
                                                       maxes + 0);
        hg->launches += 1;
        if (int rc = scan(col_deg, n, hg->col_ptr)) return rc;
        k_col_fill<<<blocks(E, 256), 256, 0, st>>>(hg->col_idx, E, hg->col_ptr, cursor, hg->col_edge);
        hg->launches += 1;
        // ascending edge id == ascending row, because the row CSR is row-major
        if (int rc = sort_segments(hg->col_edge, E, hg->col_ptr, n, maxes + 1)) return rc;
        k_bn_edges<<<blocks(E, 256), 256, 0, st>>>(hg->col_edge, E, edge_row, edge_pos, hg->row_ptr, hg->bn_edge);
        hg->launches += 1;
        CK(cudaGetLastError());
        int h_max[2] = {0, 0};
        CK(cudaMemcpyAsync(h_max, maxes, sizeof(h_max), cudaMemcpyDeviceToHost, st));
        int rc = read_err();  // synchronises
        if (rc) return rc;
        hg->max_row_deg = h_max[0];
        hg->max_col_deg = h_max[1];
        if (hg->max_row_deg > 65535) return fail(LDPC_ERR_UNSUPPORTED);
        scratch_free();
        return LDPC_OK;
    }
};

}  // namespace

void HostGraph::free_all() {
    cudaFree(row_ptr); cudaFree(col_idx); cudaFree(col_ptr); cudaFree(col_edge); cudaFree(bn_edge); cudaFree(bn_off);
    row_ptr = col_idx = col_ptr = col_edge = nullptr;
    bn_edge = nullptr;
    bn_off = nullptr;
}

int ingest_dense(const uint8_t *H, int m, int n, cudaStream_t st, HostGraph *hg) {
    Builder b{hg, st};
    auto on_error = [&] { b.on_error(); };
    hg->m = m;
    hg->n = n;
    CK(cudaMalloc(&b.row_deg, sizeof(int) * m));
    CK(cudaMalloc(&b.err, sizeof(int)));
    CK(cudaMalloc(&b.maxes, sizeof(int) * 2));
    CK(cudaMalloc(&hg->row_ptr, sizeof(int) * (m + 1)));
    CK(cudaMemsetAsync(b.err, 0, sizeof(int), st));
    CK(cudaMemsetAsync(b.maxes, 0, sizeof(int) * 2, st));
    unsigned long long *total = nullptr;
    CK(cudaMalloc(&total, sizeof(unsigned long long)));
    CK(cudaMemsetAsync(total, 0, sizeof(unsigned long long), st));
    k_dense_count<<<blocks((int64_t)m * 32, 256), 256, 0, st>>>(H, m, n, b.row_deg, b.err, total);
    hg->launches += 1;
    CK(cudaGetLastError());
    unsigned long long E64 = 0;
    CK(cudaMemcpyAsync(&E64, total, sizeof(E64), cudaMemcpyDeviceToHost, st));
    int rc = b.read_err();  // synchronises; NOT_BINARY is reported before anything else is built
    cudaFree(total);
    if (rc) return rc;
    if (E64 >= 0x7fffffffull) return b.fail(LDPC_ERR_UNSUPPORTED);
    const int E = (int)E64;
    if ((rc = b.scan(b.row_deg, m, hg->row_ptr))) return rc;
    hg->E = E;
    CK(cudaMalloc(&hg->col_idx, sizeof(int) * std::max(E, 1)));
    k_dense_fill<<<blocks((int64_t)m * 32, 256), 256, 0, st>>>(H, m, n, hg->row_ptr, hg->col_idx);
    hg->launches += 1;
    CK(cudaGetLastError());
    return b.columns();
}

int ingest_coo(const int32_t *rows, const int32_t *cols, int64_t nnz, int m, int n, cudaStream_t st,
               HostGraph *hg) {
    Builder b{hg, st};
    auto on_error = [&] { b.on_error(); };
    if (nnz >= 0x7fffffff) return LDPC_ERR_UNSUPPORTED;
    hg->m = m;
    hg->n = n;
    hg->E = (int)nnz;
    CK(cudaMalloc(&b.row_deg, sizeof(int) * m));
    CK(cudaMalloc(&b.err, sizeof(int)));
    CK(cudaMalloc(&b.maxes, sizeof(int) * 2));
    CK(cudaMalloc(&b.cursor, sizeof(int) * m));
    CK(cudaMalloc(&hg->row_ptr, sizeof(int) * (m + 1)));
    CK(cudaMalloc(&hg->col_idx, sizeof(int) * std::max<int64_t>(nnz, 1)));
    CK(cudaMemsetAsync(b.row_deg, 0, sizeof(int) * m, st));
    CK(cudaMemsetAsync(b.cursor, 0, sizeof(int) * m, st));
    CK(cudaMemsetAsync(b.err, 0, sizeof(int), st));
    CK(cudaMemsetAsync(b.maxes, 0, sizeof(int) * 2, st));
    k_coo_count<<<blocks(nnz, 256), 256, 0, st>>>(rows, cols, nnz, m, n, b.row_deg, b.err);
    hg->launches += 1;
    CK(cudaGetLastError());
    int rc = b.read_err();  // range errors first: the fill below indexes by row
    if (rc) return rc;
    if ((rc = b.scan(b.row_deg, m, hg->row_ptr))) return rc;
    k_coo_fill<<<blocks(nnz, 256), 256, 0, st>>>(rows, cols, nnz, hg->row_ptr, b.cursor, hg->col_idx);
    hg->launches += 1;
    if ((rc = b.sort_segments(hg->col_idx, (int)nnz, hg->row_ptr, m, b.maxes + 0))) return rc;
    CK(cudaGetLastError());
    cudaFree(b.cursor);
    b.cursor = nullptr;
    return b.columns();
}

}  // namespace ldpc
