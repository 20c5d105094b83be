// tools/graph_floor.cu -- the launch floor of a request graph on B200 (C5
// small-request latency): replay time of a CUDA graph of K
// dependent kernels that do (almost) nothing, with and without programmatic
// dependent launch (PDL), and of K dependent kernels that each read and write
// 512 KiB (one N = 2^16 residue row) from L2 with 148 CTAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/libs/graph_floor tools/graph_floor.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void k_empty(int* p)
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p && threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p, 1);
}

__global__ void k_touch(uint64_t* d, uint32_t words)
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < words; i += gridDim.x * blockDim.x) d[i] = d[i] * 3 + 1;
}

static cudaError_t launch(bool pdl, void (*fn)(int*), int* p, unsigned grid, cudaStream_t st)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fn, p);
}
static cudaError_t launch_touch(bool pdl, uint64_t* d, uint32_t words, cudaStream_t st)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_touch, d, words);
}

int main()
{
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    int* p;
    cudaMalloc(&p, sizeof(int));
    uint64_t* d;
    const uint32_t words = 1u << 16;
    cudaMalloc(&d, words * 8);
    cudaMemset(d, 0, words * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode)
        for (int pdl = 0; pdl < 2; ++pdl)
            for (int K : {1, 2, 4, 8}) {
                cudaGraph_t g;
                cudaGraphExec_t ge;
                cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
                for (int k = 0; k < K; ++k) {
                    if (mode == 0) launch(pdl, k_empty, p, 148, st);
                    else launch_touch(pdl, d, words, st);
                }
                cudaStreamEndCapture(st, &g);
                cudaGraphInstantiateWithFlags(&ge, g, 0);
                for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, st);
                cudaStreamSynchronize(st);
                // latency: one replay at a time
                float best = 1e9, sum = 0;
                const int reps = 200;
                for (int r = 0; r < reps; ++r) {
                    cudaEventRecord(e0, st);
                    cudaGraphLaunch(ge, st);
                    cudaEventRecord(e1, st);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    sum += ms;
                    if (ms < best) best = ms;
                }
                // back to back
                cudaEventRecord(e0, st);
                for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, st);
                cudaEventRecord(e1, st);
                cudaEventSynchronize(e1);
                float tot;
                cudaEventElapsedTime(&tot, e0, e1);
                printf("{\"kernels\": \"%s\", \"pdl\": %d, \"K\": %d, \"latency_us_mean\": %.2f, \"latency_us_min\": %.2f, "
                       "\"stream_us_per_replay\": %.2f, \"err\": \"%s\"}\n",
                       mode ? "touch 512 KiB, 148 CTAs" : "empty, 148 CTAs", pdl, K, sum / reps * 1e3, best * 1e3,
                       tot / reps * 1e3, cudaGetErrorString(cudaGetLastError()));
                cudaGraphExecDestroy(ge);
                cudaGraphDestroy(g);
            }
    return 0;
}
