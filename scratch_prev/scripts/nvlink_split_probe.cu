// nvlink_split_probe.cu -- does pushing (sender SMs store into the peer) and
// pulling (receiver SMs load from the peer) at the same time move more bytes
// over one link direction than either alone?  Single process, 2 GPUs, peer
// access; TMA bulk copies through a shared-memory ring, one elected thread
// per CTA (the same engine as kvx_bulk_kernel).  Data flows GPU1 -> GPU0 in
// every case.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_split_probe nvlink_split_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);       \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

constexpr int kStages = 4;
constexpr uint32_t kChunk = 32768;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_copy(const char* __restrict__ src, char* __restrict__ dst, uint64_t bytes) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[kStages];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < kStages; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint64_t nchunks = bytes / kChunk;
    uint32_t phase[kStages] = {0};
    uint64_t issued = 0;
    int slot = 0;
    // simple ring: load chunk i into slot i % S, wait, store; keep S loads in flight
    uint64_t c0 = blockIdx.x, step = gridDim.x;
    uint64_t inflight_c[kStages];
    int n_in = 0;
    for (uint64_t c = c0; c < nchunks || n_in > 0;) {
        if (c < nchunks && n_in < kStages) {
            // slot free once its previous store was read
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kStages - 1) : "memory");
            uint64_t* bar = &bars[slot];
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(kChunk)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(smem + (size_t)slot * kChunk)),
                "l"(src + c * kChunk), "r"(kChunk), "r"(su32(bar))
                : "memory");
            inflight_c[slot] = c;
            slot = (slot + 1) % kStages;
            ++n_in;
            c += step;
            ++issued;
            continue;
        }
        // retire the oldest
        const int old = (slot - n_in + kStages) % kStages;
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                su32(&bars[old])),
            "r"(phase[old])
            : "memory");
        phase[old] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + inflight_c[old] * kChunk),
                     "r"(su32(smem + (size_t)old * kChunk)), "r"(kChunk)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        --n_in;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __threadfence_system();
}

int main() {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < 2) {
        printf("needs 2 GPUs\n");
        return 1;
    }
    const uint64_t bytes = 4ull << 30;  // per direction per mover
    char *g0_dst_push, *g0_dst_pull, *g1_src_push, *g1_src_pull;
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    CK(cudaMalloc(&g0_dst_push, bytes));
    CK(cudaMalloc(&g0_dst_pull, bytes));
    CK(cudaFuncSetAttribute(bulk_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk));
    CK(cudaSetDevice(1));
    CK(cudaDeviceEnablePeerAccess(0, 0));
    CK(cudaMalloc(&g1_src_push, bytes));
    CK(cudaMalloc(&g1_src_pull, bytes));
    CK(cudaMemset(g1_src_push, 1, bytes));
    CK(cudaMemset(g1_src_pull, 2, bytes));
    CK(cudaFuncSetAttribute(bulk_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk));
    cudaStream_t s0, s1;
    CK(cudaSetDevice(0));
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaSetDevice(1));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    // ---- bidirectional: both link directions loaded at once
    {
        char *g0_src, *g1_dst, *g0_dst2, *g1_src2;
        CK(cudaSetDevice(0));
        CK(cudaMalloc(&g0_src, bytes));
        CK(cudaMemset(g0_src, 3, bytes));
        CK(cudaSetDevice(1));
        CK(cudaMalloc(&g1_dst, bytes));
        (void)g0_dst2;
        (void)g1_src2;
        const char* names[] = {"bi_push", "bi_pull", "bi_push01_pull10", "bi_copy_engine", "bi_half_push_half_pull"};
        cudaStream_t s0b, s1b;
        CK(cudaSetDevice(0));
        CK(cudaStreamCreateWithFlags(&s0b, cudaStreamNonBlocking));
        CK(cudaSetDevice(1));
        CK(cudaStreamCreateWithFlags(&s1b, cudaStreamNonBlocking));
        for (int ctas : {64, 148}) {
            for (int mode = 0; mode < 5; ++mode) {
                if (mode == 2) continue;  // superseded by mode 4
                double best = 1e30;
                for (int rep = 0; rep < 4; ++rep) {
                    CK(cudaSetDevice(0));
                    CK(cudaDeviceSynchronize());
                    CK(cudaSetDevice(1));
                    CK(cudaDeviceSynchronize());
                    cudaEvent_t a, b, done1;
                    CK(cudaSetDevice(0));
                    CK(cudaEventCreate(&a));
                    CK(cudaEventCreate(&b));
                    CK(cudaSetDevice(1));
                    CK(cudaEventCreateWithFlags(&done1, cudaEventDisableTiming));
                    CK(cudaSetDevice(0));
                    CK(cudaEventRecord(a, s0));
                    CK(cudaSetDevice(1));
                    CK(cudaStreamWaitEvent(s1, a, 0));
                    // direction 1->0 (g1_src_push -> g0_dst_push) and 0->1 (g0_src -> g1_dst)
                    if (mode == 0) {  // each GPU pushes its outgoing data
                        bulk_copy<<<ctas, 32, kStages * kChunk, s1>>>(g1_src_push, g0_dst_push, bytes);
                    } else if (mode == 1) {  // each GPU pulls its incoming data
                        bulk_copy<<<ctas, 32, kStages * kChunk, s1>>>(g0_src, g1_dst, bytes);
                    } else if (mode == 2) {  // GPU0 pushes 0->1 and pulls 1->0; GPU1 idle
                    } else if (mode == 4) {  // each direction: half pushed by its sender, half pulled by its receiver
                        const uint64_t h = bytes / 2;
                        // GPU1: push first half of 1->0, pull second half of 0->1
                        CK(cudaStreamWaitEvent(s1b, a, 0));
                        bulk_copy<<<ctas / 2, 32, kStages * kChunk, s1>>>(g1_src_push, g0_dst_push, h);
                        bulk_copy<<<ctas / 2, 32, kStages * kChunk, s1b>>>(g0_src + h, g1_dst + h, h);
                        cudaEvent_t j1;
                        CK(cudaEventCreateWithFlags(&j1, cudaEventDisableTiming));
                        CK(cudaEventRecord(j1, s1b));
                        CK(cudaStreamWaitEvent(s1, j1, 0));
                        CK(cudaEventDestroy(j1));
                    } else {
                        CK(cudaMemcpyPeerAsync(g0_dst_push, 0, g1_src_push, 1, bytes, s1));
                    }
                    CK(cudaEventRecord(done1, s1));
                    CK(cudaSetDevice(0));
                    if (mode == 0) {
                        bulk_copy<<<ctas, 32, kStages * kChunk, s0>>>(g0_src, g1_dst, bytes);
                    } else if (mode == 1) {
                        bulk_copy<<<ctas, 32, kStages * kChunk, s0>>>(g1_src_pull, g0_dst_pull, bytes);
                    } else if (mode == 2) {
                        bulk_copy<<<ctas / 2, 32, kStages * kChunk, s0>>>(g0_src, g1_dst, bytes);
                        bulk_copy<<<ctas / 2, 32, kStages * kChunk, s0>>>(g1_src_pull, g0_dst_pull, bytes);
                    } else if (mode == 4) {  // GPU0: push first half of 0->1, pull second half of 1->0
                        const uint64_t h = bytes / 2;
                        CK(cudaStreamWaitEvent(s0b, a, 0));
                        bulk_copy<<<ctas / 2, 32, kStages * kChunk, s0>>>(g0_src, g1_dst, h);
                        bulk_copy<<<ctas / 2, 32, kStages * kChunk, s0b>>>(g1_src_push + h, g0_dst_push + h, h);
                        cudaEvent_t j0;
                        CK(cudaEventCreateWithFlags(&j0, cudaEventDisableTiming));
                        CK(cudaEventRecord(j0, s0b));
                        CK(cudaStreamWaitEvent(s0, j0, 0));
                        CK(cudaEventDestroy(j0));
                    } else {
                        CK(cudaMemcpyPeerAsync(g1_dst, 1, g0_src, 0, bytes, s0));
                    }
                    CK(cudaStreamWaitEvent(s0, done1, 0));
                    CK(cudaEventRecord(b, s0));
                    CK(cudaEventSynchronize(b));
                    CK(cudaGetLastError());
                    float ms = 0;
                    CK(cudaEventElapsedTime(&ms, a, b));
                    if (rep) best = ms < best ? ms : best;
                    if (rep == 3)
                        printf("{\"ctas\": %d, \"mode\": \"%s\", \"GBps_per_direction\": %.1f, \"ms\": %.3f}\n",
                               ctas, names[mode], (double)bytes / (best * 1e-3) / 1e9, best);
                    CK(cudaEventDestroy(a));
                    CK(cudaEventDestroy(b));
                    CK(cudaSetDevice(1));
                    CK(cudaEventDestroy(done1));
                }
            }
        }
    }
    int ctas_list[] = {16, 32, 64, 148};
    for (int ctas : ctas_list) {
        for (int mode = 0; mode < 4; ++mode) {  // 0 push, 1 pull, 2 push+pull, 3 copy engine
            double best = 1e30;
            for (int rep = 0; rep < 4; ++rep) {
                CK(cudaSetDevice(0));
                CK(cudaDeviceSynchronize());
                CK(cudaSetDevice(1));
                CK(cudaDeviceSynchronize());
                cudaEvent_t a, b;
                CK(cudaSetDevice(0));
                CK(cudaEventCreate(&a));
                CK(cudaEventCreate(&b));
                const uint64_t part = mode == 2 ? bytes / 2 : bytes;
                // events on GPU0's stream; GPU1's work joins through a wait
                cudaEvent_t done1;
                CK(cudaSetDevice(1));
                CK(cudaEventCreateWithFlags(&done1, cudaEventDisableTiming));
                CK(cudaSetDevice(0));
                CK(cudaEventRecord(a, s0));
                CK(cudaSetDevice(1));
                CK(cudaStreamWaitEvent(s1, a, 0));
                if (mode == 0 || mode == 2)  // GPU1 SMs store into GPU0
                    bulk_copy<<<ctas, 32, kStages * kChunk, s1>>>(g1_src_push, g0_dst_push, part);
                if (mode == 3) CK(cudaMemcpyPeerAsync(g0_dst_push, 0, g1_src_push, 1, part, s1));
                CK(cudaEventRecord(done1, s1));
                CK(cudaSetDevice(0));
                if (mode == 1 || mode == 2)  // GPU0 SMs load from GPU1
                    bulk_copy<<<ctas, 32, kStages * kChunk, s0>>>(g1_src_pull, g0_dst_pull, part);
                CK(cudaStreamWaitEvent(s0, done1, 0));
                CK(cudaEventRecord(b, s0));
                CK(cudaEventSynchronize(b));
                CK(cudaGetLastError());
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, a, b));
                const double moved = mode == 2 ? (double)part * 2 : (double)part;
                if (rep) best = ms < best ? ms : best;
                if (rep == 3)
                    printf("{\"ctas\": %d, \"mode\": \"%s\", \"GBps\": %.1f, \"ms\": %.3f}\n", ctas,
                           mode == 0 ? "push" : mode == 1 ? "pull" : mode == 2 ? "push+pull" : "copy_engine",
                           moved / (best * 1e-3) / 1e9, best);
                CK(cudaEventDestroy(a));
                CK(cudaEventDestroy(b));
                CK(cudaSetDevice(1));
                CK(cudaEventDestroy(done1));
            }
        }
    }
    return 0;
}
