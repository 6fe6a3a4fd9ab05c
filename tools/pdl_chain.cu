// Microbenchmark (dev tool): cost of one link of a programmatic-dependent-launch
// chain of near-empty kernels on B200, by grid size, with and without PDL —
// the fixed per-launch cost behind the frame's 31 kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/pdl_chain.cu -o /tmp/pc && /tmp/pc
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void k_link(int* x, int trigger_early) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (trigger_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) atomicAdd(x + (blockIdx.x & 63), 1);
}

int main() {
    int* x;
    cudaMalloc(&x, 64 * sizeof(int));
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int N = 2000;
    for (int pdl = 0; pdl < 2; ++pdl)
        for (int trig = 0; trig < 2; ++trig)
            for (int grid : {32, 148, 296, 1184}) {
                if (!pdl && trig) continue;
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cfg.attrs = attr;
                cfg.numAttrs = pdl ? 1 : 0;
                for (int w = 0; w < 100; ++w) cudaLaunchKernelEx(&cfg, k_link, x, trig);
                cudaEventRecord(a, s);
                for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, k_link, x, trig);
                cudaEventRecord(b, s);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                // the same chain as one CUDA graph (no host launch cost inside the timed region)
                cudaGraph_t gph;
                cudaGraphExec_t ge;
                cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
                for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, k_link, x, trig);
                cudaStreamEndCapture(s, &gph);
                cudaGraphInstantiate(&ge, gph, 0);
                cudaGraphLaunch(ge, s);
                cudaEventRecord(a, s);
                cudaGraphLaunch(ge, s);
                cudaEventRecord(b, s);
                cudaEventSynchronize(b);
                float mg;
                cudaEventElapsedTime(&mg, a, b);
                cudaGraphExecDestroy(ge);
                cudaGraphDestroy(gph);
                printf("pdl %d trigger %d grid %5d x 256: %.2f us per link (stream), %.2f us (graph)\n", pdl, trig, grid,
                       ms * 1e3 / N, mg * 1e3 / N);
            }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
