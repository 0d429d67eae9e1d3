// L2 -> SM bandwidth ceiling on this GPU (the bound of the streaming bit node, whose row-record gathers
// hit L2): every warp reads 512-byte float4 segments of an L2-resident buffer (32 MB, read repeatedly;
// the segment order is a fixed pseudo-random permutation, like the bit node's gathers), persistent grid
// of 148 x 12 CTAs of 128 threads.  Prints GB/s of bytes delivered to the SMs.  Also a DRAM stream
// (4 GB buffer, read once per pass) for the HBM read figure under the same access pattern.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(128, 12) gather(const float4 *__restrict__ buf, int nseg, int iters,
                                                  unsigned mul, float *out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int it = 0; it < iters; it++) {
        for (int s = warp; s < nseg; s += nw) {
            const unsigned seg = ((unsigned)s * mul + (unsigned)it) & (unsigned)(nseg - 1);  // permutation (nseg = 2^k)
            const float4 v = __ldg(buf + (size_t)seg * 32 + lane);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    if (acc.x == 12345.f) out[0] = acc.y + acc.z + acc.w;
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, 4);
    const size_t sizes[2] = {(size_t)32 << 20, (size_t)4 << 30};
    const int iters[2] = {64, 2};
    for (int q = 0; q < 2; q++) {
        float4 *buf;
        cudaMalloc(&buf, sizes[q]);
        cudaMemset(buf, 0, sizes[q]);
        const int nseg = (int)(sizes[q] / 512);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        gather<<<sms * 12, 128>>>(buf, nseg, 2, 2654435761u, out);  // warm
        cudaEventRecord(a);
        gather<<<sms * 12, 128>>>(buf, nseg, iters[q], 2654435761u, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)nseg * 512.0 * iters[q];
        printf("{\"what\": \"%s\", \"buffer_bytes\": %zu, \"GBps\": %.1f}\n",
               q == 0 ? "L2-resident 512-byte segment gathers" : "DRAM 512-byte segment gathers", sizes[q],
               bytes / ms / 1e6);
        cudaFree(buf);
    }
    return 0;
}
