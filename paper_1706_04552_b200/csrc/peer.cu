// peer.cu -- halo exchange of the partitioned CA over peer memory:
// no NCCL call per step.  Every rank maps its peers' ping-pong buffers and flag
// words once (CUDA IPC; over NVLink/NVSwitch on a multi-GPU box, plain device
// memory when two processes share one GPU, which is how the tests run it).
//
// After a rank's step kernel has written state t+1 into its dst buffer:
//   put  : one CTA copies the rank's changing halo cells (PartitionPlan.exchange_slots,
//          a few hundred cells) from its own dst into every peer's dst at the same
//          linear indices (peers never write cells they do not own), then
//          __threadfence_system() and a release store of `epoch` into the rank's slot
//          of every peer's flag array;
//   wait : before step t+1 reads dst, one thread acquires every peer's slot in its
//          own flag array until it reaches `epoch` (bounded: after ~`timeout_ns` it
//          records GM_PEER_TIMEOUT in a status word instead of hanging the GPU).
// Ordering argument (why one flag per step is enough): a rank starts step t+1 only
// after every peer signalled step t, i.e. finished reading the buffer the rank's
// step-t+1 put will write into.
#include <cstdint>

#include "launch.h"

namespace gm {
namespace {

template <int C>
struct CellT;
template <> struct CellT<1> { using T = uint8_t; };
template <> struct CellT<2> { using T = uint16_t; };
template <> struct CellT<4> { using T = uint32_t; };
template <> struct CellT<8> { using T = uint64_t; };

template <int C>
__global__ void peer_put(const uint8_t* __restrict__ mine, const uint64_t* __restrict__ peers,
                         const int64_t* __restrict__ idx, const int64_t* __restrict__ didx, int64_t k,
                         const uint64_t* __restrict__ peer_flags, int rank, int world, uint64_t epoch) {
    using T = typename CellT<C>::T;
    const T* src = reinterpret_cast<const T*>(mine);
    if (didx != nullptr) {  // tiled storage: per entry the destination rank (bits 56-63) and cell
        for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
            const uint64_t d = (uint64_t)didx[i];
            const int q = (int)(d >> 56);
            T* dst = q == rank ? const_cast<T*>(src) : reinterpret_cast<T*>(peers[q]);
            dst[d & ((1ull << 56) - 1)] = src[idx[i]];
        }
    } else {
        for (int q = 0; q < world; ++q) {
            if (q == rank) continue;
            T* dst = reinterpret_cast<T*>(peers[q]);
            for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
                const int64_t c = idx[i];
                dst[c] = src[c];
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();  // the cells reach every peer before its flag does
        for (int q = 0; q < world; ++q) {
            if (q == rank) continue;
            uint64_t* f = reinterpret_cast<uint64_t*>(peer_flags[q]) + rank;
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
        }
    }
}

__global__ void peer_wait(const uint64_t* flags, int rank, int world, uint64_t epoch, uint64_t timeout_ns,
                          uint32_t* status) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int p = 0; p < world; ++p) {
        if (p == rank) continue;
        for (;;) {
            uint64_t v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + p) : "memory");
            if (v >= epoch) break;
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) {
                atomicOr(status, 1u << (p & 31));
                return;
            }
            __nanosleep(200);
        }
    }
}

}  // namespace

cudaError_t launch_peer_put(const void* mine, const uint64_t* peers, const int64_t* idx, const int64_t* didx,
                            int64_t k, int cell_bytes, const uint64_t* peer_flags, int rank, int world, uint64_t epoch,
                            cudaStream_t s) {
    const auto* m = reinterpret_cast<const uint8_t*>(mine);
    switch (cell_bytes) {
    case 1: peer_put<1><<<1, 256, 0, s>>>(m, peers, idx, didx, k, peer_flags, rank, world, epoch); break;
    case 2: peer_put<2><<<1, 256, 0, s>>>(m, peers, idx, didx, k, peer_flags, rank, world, epoch); break;
    case 4: peer_put<4><<<1, 256, 0, s>>>(m, peers, idx, didx, k, peer_flags, rank, world, epoch); break;
    case 8: peer_put<8><<<1, 256, 0, s>>>(m, peers, idx, didx, k, peer_flags, rank, world, epoch); break;
    default: return cudaErrorInvalidValue;
    }
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_peer_wait(const uint64_t* flags, int rank, int world, uint64_t epoch, uint64_t timeout_ns,
                             uint32_t* status, cudaStream_t s) {
    peer_wait<<<1, 1, 0, s>>>(flags, rank, world, epoch, timeout_ns, status);
    note_launch();
    return cudaGetLastError();
}

}  // namespace gm
