// ingest.cu -- RatingsMatrix::from_triplets (sparse.hpp:73-149) on the GPU.
//
// The reference validates the triplets in input order (first offending one decides the error), then
// builds the CSR with a stable two-pass counting sort (by column, then by row), rejects the first
// duplicate in row order, and mirrors the CSC from the CSR so every column's rows ascend.  Here: one
// pass packs (user, item) into a 64-bit key (user above item, only as many bits as m and n need) and
// records the first invalid triplet with an atomicMin over its index; a stable radix sort by key
// (CUB onesweep) gives the CSR order; one pass finds the first duplicate (adjacent equal keys, in
// row order = sorted order), writes the column indices and the row offsets; the CSC is the same with
// (item, user) keys.  The output is bitwise the reference's (same order, same values).
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device.hpp"

namespace pmfgpu {

namespace {

__global__ void pack_kernel(const DevTriplet* __restrict__ t, int64_t nnz, int32_t m, int32_t n, int bits_minor,
                            bool item_minor, unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals,
                            unsigned long long* __restrict__ first_bad) {
    for (int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < nnz;
         x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const DevTriplet v = t[x];
        const bool bad = v.user < 0 || v.user >= m || v.item < 0 || v.item >= n || !isfinite(v.rating);
        if (bad) atomicMin(first_bad, static_cast<unsigned long long>(x));
        const uint64_t major = static_cast<uint32_t>(item_minor ? v.user : v.item);
        const uint64_t minor = static_cast<uint32_t>(item_minor ? v.item : v.user);
        keys[x] = bad ? 0ull : (major << bits_minor) | minor;
        vals[x] = __float_as_uint(v.rating);
    }
}

// Sorted keys -> minor indices, major offsets start[0..count], first duplicate position.
__global__ void offsets_kernel(const unsigned long long* __restrict__ keys, int64_t nnz, int bits_minor,
                               int32_t count, int64_t* __restrict__ start, int32_t* __restrict__ minor_out,
                               unsigned long long* __restrict__ first_dup) {
    const uint64_t mask = (uint64_t(1) << bits_minor) - 1;
    for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p <= nnz;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t cur = p < nnz ? static_cast<int64_t>(keys[p] >> bits_minor) : count;
        const int64_t prev = p > 0 ? static_cast<int64_t>(keys[p - 1] >> bits_minor) : -1;
        for (int64_t r = prev + 1; r <= cur; ++r) start[r] = p;  // majors prev+1 .. cur start at p
        if (p < nnz) {
            minor_out[p] = static_cast<int32_t>(keys[p] & mask);
            if (p > 0 && keys[p] == keys[p - 1]) atomicMin(first_dup, static_cast<unsigned long long>(p));
        }
    }
}

int bits_for(int32_t count) {
    int b = 1;
    while (b < 31 && (int64_t(1) << b) < count) ++b;
    return b;
}

}  // namespace

// Builds CSR + CSC of `nnz` device triplets into device arrays.  Returns in *bad the index of the
// first invalid triplet (or -1), in *dup the CSR position of the first duplicate (or -1); the
// outputs are valid only when both are -1.  scratch: caller-owned device memory of
// ingest_scratch_bytes(nnz) bytes.
size_t ingest_scratch_bytes(int64_t nnz) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<const unsigned long long*>(nullptr),
                                    static_cast<unsigned long long*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<int>(nnz), 0, 62);
    const size_t n = static_cast<size_t>(nnz > 0 ? nnz : 1);
    return 2 * n * sizeof(unsigned long long) + 2 * n * sizeof(uint32_t) + 2 * sizeof(unsigned long long) +
           ((temp + 255) & ~size_t(255)) + 1024;
}

#define INGEST_TRY(x)                     \
    do {                                  \
        const cudaError_t e_ = (x);       \
        if (e_ != cudaSuccess) return e_; \
    } while (0)

cudaError_t ingest_build(const DevTriplet* t, int64_t nnz, int32_t m, int32_t n, void* scratch, int64_t* row_start,
                  int32_t* col_of, float* val_row, int64_t* col_start, int32_t* row_of, float* val_col,
                  int64_t* bad, int64_t* dup, cudaStream_t s) {
    const size_t N = static_cast<size_t>(nnz > 0 ? nnz : 1);
    char* p = static_cast<char*>(scratch);
    auto* k0 = reinterpret_cast<unsigned long long*>(p);
    auto* k1 = k0 + N;
    auto* v0 = reinterpret_cast<uint32_t*>(k1 + N);
    auto* v1 = v0 + N;
    auto* flags = reinterpret_cast<unsigned long long*>(
        (reinterpret_cast<uintptr_t>(v1 + N) + 255) & ~uintptr_t(255));  // [0] first bad, [1] first dup
    void* temp = flags + 32;
    size_t temp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, k0, k1, v0, v1, static_cast<int>(nnz), 0, 62, s);
    const int threads = 256;
    const int blocks = static_cast<int>(std::min<int64_t>((nnz + threads) / threads + 1, 148 * 16));
    unsigned long long h[2];
    for (int side = 0; side < 2; ++side) {
        const bool csr = side == 0;
        const int bits_minor = bits_for(csr ? n : m);
        const int bits_major = bits_for(csr ? m : n);
        INGEST_TRY(cudaMemsetAsync(flags, 0xff, 2 * sizeof(unsigned long long), s));
        pack_kernel<<<blocks, threads, 0, s>>>(t, nnz, m, n, bits_minor, csr, k0, v0, flags);
        if (csr) {
            INGEST_TRY(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s));
            INGEST_TRY(cudaStreamSynchronize(s));
            if (h[0] != ~0ull) {
                *bad = static_cast<int64_t>(h[0]);
                *dup = -1;
                return cudaSuccess;
            }
        }
        if (nnz > 0)
            INGEST_TRY(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k0, k1, v0, v1, static_cast<int>(nnz), 0,
                                                       bits_minor + bits_major, s));
        offsets_kernel<<<blocks, threads, 0, s>>>(k1, nnz, bits_minor, csr ? m : n, csr ? row_start : col_start,
                                                  csr ? col_of : row_of, flags + 1);
        INGEST_TRY(cudaMemcpyAsync(csr ? static_cast<void*>(val_row) : static_cast<void*>(val_col), v1,
                                         static_cast<size_t>(nnz) * sizeof(float), cudaMemcpyDeviceToDevice, s));
        if (csr) {
            INGEST_TRY(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s));
            INGEST_TRY(cudaStreamSynchronize(s));
            if (h[1] != ~0ull) {
                *bad = -1;
                *dup = static_cast<int64_t>(h[1]);
                return cudaSuccess;
            }
        }
    }
    INGEST_TRY(cudaGetLastError());
    *bad = -1;
    *dup = -1;
    return cudaSuccess;
}

}  // namespace pmfgpu
