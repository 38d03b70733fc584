// peer_epilogue.cuh -- the partitioned CA's halo exchange fused into the step kernel
// (`gm_run_part_peer`): the kernel that computes state t+1 also moves
// it to the peers, over peer memory, with no separate launch and no collective.
//
//   prologue : thread 0 of every CTA acquires the peers' step flags (>= wait_epoch:
//              their halo cells of the state this kernel reads have landed), bounded;
//   epilogue : every CTA fences its stores and bumps a grid-wide counter; the last CTA
//              copies the rank's changing halo cells from its new state into every
//              peer's new-state buffer, fences system-wide and release-stores
//              signal_epoch into the rank's slot of every peer's flag array.
// Same protocol as peer.cu's put/wait kernels (see there for the ordering argument).
#pragma once
#include <cstdint>

#define GM_MAX_PEERS 16

namespace gm {

struct PeerEpilogue {
    uint64_t peers[GM_MAX_PEERS];       // new-state buffer of every rank (this parity)
    uint64_t peer_flags[GM_MAX_PEERS];  // flag array of every rank
    uint64_t own_flags;                 // this rank's flag array
    uint64_t idx;                       // const int64_t*: the rank's halo cells (linear)
    int64_t count;
    int32_t cell_bytes, rank, world;
    uint32_t done;                      // CTAs finished in the current launch
    uint32_t status;                    // bit p: waiting on peer p timed out
    uint64_t didx;                      // const int64_t*: tiled storage: per entry, the destination
                                        // cell (bits 0-55) and rank (bits 56-63; own rank = a ring
                                        // copy inside this rank's buffer); 0 = every peer, same index
};

constexpr int PEER_RANK_SHIFT = 56;

__device__ __forceinline__ void peer_prologue_wait(PeerEpilogue* e, uint64_t epoch) {
    if (e == nullptr || epoch == 0) return;
    if (threadIdx.x == 0) {
        const uint64_t* flags = reinterpret_cast<const uint64_t*>(e->own_flags);
        uint64_t t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (int p = 0; p < e->world; ++p) {
            if (p == e->rank) continue;
            for (;;) {
                uint64_t v;
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + p) : "memory");
                if (v >= epoch) break;
                uint64_t t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t - t0 > 10000000000ull) {  // 10 s: record, do not hang the GPU
                    atomicOr(&e->status, 1u << (p & 31));
                    break;
                }
                __nanosleep(256);
            }
        }
    }
    __syncthreads();
}

template <class T>
__device__ __forceinline__ void peer_copy_cells(const uint8_t* grid, PeerEpilogue* e) {
    const int64_t* idx = reinterpret_cast<const int64_t*>(e->idx);
    const T* src = reinterpret_cast<const T*>(grid);
    if (e->didx != 0) {  // tiled storage: (source cell, destination rank + cell) entries
        const int64_t* didx = reinterpret_cast<const int64_t*>(e->didx);
        for (int64_t i = threadIdx.x; i < e->count; i += blockDim.x) {
            const uint64_t d = (uint64_t)didx[i];
            const int q = (int)(d >> PEER_RANK_SHIFT);
            T* dst = q == e->rank ? const_cast<T*>(src) : reinterpret_cast<T*>(e->peers[q]);
            dst[d & ((1ull << PEER_RANK_SHIFT) - 1)] = src[idx[i]];
        }
        return;
    }
    for (int q = 0; q < e->world; ++q) {
        if (q == e->rank) continue;
        T* dst = reinterpret_cast<T*>(e->peers[q]);
        for (int64_t i = threadIdx.x; i < e->count; i += blockDim.x) dst[idx[i]] = src[idx[i]];
    }
}

__device__ __forceinline__ void peer_epilogue_signal(const uint8_t* grid, PeerEpilogue* e, uint64_t epoch) {
    if (e == nullptr || epoch == 0) return;
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();  // this CTA's stores before the count
        last = atomicAdd(&e->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();  // every CTA's stores are visible to the last one
    switch (e->cell_bytes) {
    case 1: peer_copy_cells<uint8_t>(grid, e); break;
    case 2: peer_copy_cells<uint16_t>(grid, e); break;
    case 4: peer_copy_cells<uint32_t>(grid, e); break;
    default: peer_copy_cells<uint64_t>(grid, e); break;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();  // the cells reach every peer before its flag does
        for (int q = 0; q < e->world; ++q) {
            if (q == e->rank) continue;
            uint64_t* f = reinterpret_cast<uint64_t*>(e->peer_flags[q]) + e->rank;
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
        }
        e->done = 0;  // ready for the next launch with this descriptor
    }
}

}  // namespace gm
