// Microbenchmarks: cooperative-groups grid.sync vs a hand-rolled grid
// barrier, and the last-block (ticket) reduction pattern.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned long long* out) {
    cg::grid_group g = cg::this_grid();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

// sense-reversing barrier: one arrival counter per barrier generation
__device__ __forceinline__ void my_barrier(unsigned int* count, volatile unsigned int* gen, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int g0 = *gen;
        __threadfence();
        unsigned int a = atomicAdd(count, 1u);
        if (a == nblocks - 1) {
            *count = 0;
            __threadfence();
            *gen = g0 + 1;
        } else {
            while (*gen == g0) { __nanosleep(20); }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void k_my(int iters, unsigned int* count, unsigned int* gen, unsigned long long* out) {
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) my_barrier(count, gen, gridDim.x);
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__device__ __forceinline__ void my_barrier_spin(unsigned int* count, volatile unsigned int* gen, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int g0 = *gen;
        __threadfence();
        unsigned int a = atomicAdd(count, 1u);
        if (a == nblocks - 1) {
            *count = 0;
            __threadfence();
            *gen = g0 + 1;
        } else {
            while (*gen == g0) {}
        }
        __threadfence();
    }
    __syncthreads();
}
__global__ void k_spin(int iters, unsigned int* count, unsigned int* gen, unsigned long long* out) {
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) my_barrier_spin(count, gen, gridDim.x);
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__global__ void k_ticket(int iters, unsigned int* ticket, double* vals, unsigned long long* out) {
    cg::grid_group g = cg::this_grid();
    __shared__ int last;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) {
            vals[blockIdx.x] = i;
            __threadfence();
            unsigned int t = atomicAdd(ticket, 1u);
            last = (t == gridDim.x - 1);
        }
        __syncthreads();
        if (last) {
            __threadfence();
            double s = 0;
            for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) s += __ldcg(&vals[b]);
            if (threadIdx.x == 0) *ticket = 0;
        }
        g.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int nsm = p.multiProcessorCount;
    unsigned long long* d_out;
    unsigned int *cnt, *gen;
    double* vals;
    cudaMalloc(&d_out, 8);
    cudaMalloc(&cnt, 4);
    cudaMalloc(&gen, 4);
    cudaMalloc(&vals, 8 * 4096);
    cudaMemset(cnt, 0, 4);
    cudaMemset(gen, 0, 4);
    int iters = 2000;
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    for (int bpsm : {1, 2}) for (int threads : {256, 512}) {
        int blocks = nsm * bpsm;
        void* args[] = {&iters, &d_out};
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaLaunchCooperativeKernel((void*)k_cg, blocks, threads, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_cg, blocks, threads, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("cg grid.sync     blocks=%d threads=%d: %.3f us/sync (%s)\n", blocks, threads, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
        void* args2[] = {&iters, &cnt, &gen, &d_out};
        cudaLaunchCooperativeKernel((void*)k_my, blocks, threads, args2, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_my, blocks, threads, args2, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("custom barrier   blocks=%d threads=%d: %.3f us/sync (%s)\n", blocks, threads, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
        cudaLaunchCooperativeKernel((void*)k_spin, blocks, threads, args2, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_spin, blocks, threads, args2, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("custom spin      blocks=%d threads=%d: %.3f us/sync (%s)\n", blocks, threads, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
        void* args3[] = {&iters, &cnt, &vals, &d_out};
        cudaMemset(cnt, 0, 4);
        cudaLaunchCooperativeKernel((void*)k_ticket, blocks, threads, args3, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_ticket, blocks, threads, args3, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("ticket+grid.sync blocks=%d threads=%d: %.3f us/iter (%s)\n", blocks, threads, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
