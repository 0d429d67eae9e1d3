// synccheck probe: the persistent work-counter loop of the streaming sweeps in isolation (two CTA
// barriers per item, a divergent per-lane branch before them), to tell a tool report from a real one.
#include <cstdio>
__global__ void k(int *ctr, int items, int *out, int variant) {
    __shared__ int s_item;
    const int lane = threadIdx.x & 31;
    for (;;) {
        if (variant) __syncwarp();
        __syncthreads();
        if (threadIdx.x == 0) s_item = atomicAdd(ctr, 1);
        __syncthreads();
        const int it = s_item;
        if (it >= items) break;
        int v = 0;
        if (lane < 5) v = out[it % 7 + lane];  // per-lane branch, reconverges before the next barrier
        v = __shfl_sync(0xffffffffu, v, 0);
        if (threadIdx.x == 0) atomicAdd(out + 64, v);
    }
}
int main() {
    int *ctr, *out;
    cudaMalloc(&ctr, 4);
    cudaMalloc(&out, 65 * 4);
    cudaMemset(out, 0, 65 * 4);
    for (int variant = 0; variant < 2; variant++) {
        cudaMemset(ctr, 0, 4);
        k<<<8, 256>>>(ctr, 40, out, variant);
        printf("variant %d: %s\n", variant, cudaGetErrorString(cudaDeviceSynchronize()));
    }
    return 0;
}
