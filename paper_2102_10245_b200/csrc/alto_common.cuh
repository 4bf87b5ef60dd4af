// alto_common.cuh — shared device/host helpers for libalto_b200.so.
//
// Key/coordinate codec.  The reference decodes one bit per Python-level pass
// (layout.py:155-159, :166-168).  Here both directions are table driven:
//  * encode (deposit): for mode n and coordinate byte k, ENC[n][k][b] is the
//    key with the 8 bits of b dropped into mode n's positions g=8k..8k+7;
//    a key is the OR of ceil(b_n/8) lookups per mode.
//  * decode (extract): for key byte j, DEC[j][b] is a *packed coordinate
//    word* holding, for every mode, the coordinate bits carried by that key
//    byte, already shifted to the mode's field (mode n occupies packed bits
//    [pack_off[n], pack_off[n]+b_n), pack_off[n] = sum_{m<n} b_m).  One
//    lookup per key byte yields all modes at once; fields never overlap, so
//    OR composes.  Key bytes at or above total_bits are never read, and bits
//    >= total_bits inside the last byte map to zero, so flag bits are
//    ignored exactly as layout.py:125 requires.
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>
#include <cuda_runtime.h>

#include "../../include/alto_b200.h"

namespace alto {

// Layout digest passed by value to kernels.
struct DevLayout {
  int order, n_words, total_bits, pad_;
  int bits[ALTO_MAX_ORDER];
  int pack_off[ALTO_MAX_ORDER];
  long long dims[ALTO_MAX_ORDER];
  int enc_off[ALTO_MAX_ORDER];    // first table entry of mode n's encode tables
  int enc_bytes[ALTO_MAX_ORDER];  // ceil(bits[n]/8)
  int dec_off;                    // first entry of decode tables
  int dec_bytes;                  // ceil(total_bits/8)
  int n_entries;                  // total entries (each n_words uint64)
  int pad2_;
};

DevLayout make_dev_layout(const alto_layout* lay);

// --- error plumbing -------------------------------------------------------
void set_error(const std::string& msg);
int cuda_status(cudaError_t e, const char* where);

#define ALTO_CUDA_TRY(expr)                                          \
  do {                                                               \
    cudaError_t e__ = (expr);                                        \
    if (e__ != cudaSuccess) return ::alto::cuda_status(e__, #expr);  \
  } while (0)

#define ALTO_LAUNCH_CHECK(where)                                     \
  do {                                                               \
    cudaError_t e__ = cudaGetLastError();                            \
    if (e__ != cudaSuccess) return ::alto::cuda_status(e__, where);  \
  } while (0)

#define ALTO_REQUIRE(cond, msg)                                      \
  do {                                                               \
    if (!(cond)) { ::alto::set_error(msg); return ALTO_EINVAL; }     \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kSMs = 148;

inline int grid_for(long long n, int block, int max_blocks = kSMs * 16) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return static_cast<int>(g);
}

// --- device codec ---------------------------------------------------------

template <int W>
struct Key {
  uint64_t w[W];
};

template <int W>
__device__ __forceinline__ Key<W> load_key(const uint64_t* __restrict__ keys, long long i) {
  Key<W> k;
  if constexpr (W == 1) {
    k.w[0] = __ldg(keys + i);
  } else {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(keys) + i);
    k.w[0] = v.x;
    k.w[1] = v.y;
  }
  return k;
}

template <int W>
__device__ __forceinline__ Key<W> load_key_smem(const uint64_t* keys, int i) {
  Key<W> k;
  if constexpr (W == 1) {
    k.w[0] = keys[i];
  } else {
    const ulonglong2 v = reinterpret_cast<const ulonglong2*>(keys)[i];
    k.w[0] = v.x;
    k.w[1] = v.y;
  }
  return k;
}

template <int W>
__device__ __forceinline__ void store_key(uint64_t* keys, long long i, const Key<W>& k) {
  if constexpr (W == 1) {
    keys[i] = k.w[0];
  } else {
    reinterpret_cast<ulonglong2*>(keys)[i] = make_ulonglong2(k.w[0], k.w[1]);
  }
}

// Packed coordinate word from a key: OR of one table entry per key byte.
// `tab` points at the decode tables (entry 0 = key byte 0, value 0).
template <int W>
__device__ __forceinline__ Key<W> decode_packed(const uint64_t* __restrict__ tab, int dec_bytes,
                                                const Key<W>& k) {
  Key<W> p;
#pragma unroll
  for (int i = 0; i < W; ++i) p.w[i] = 0;
#pragma unroll
  for (int j = 0; j < 8 * W; ++j) {
    if (j < dec_bytes) {
      const unsigned b = static_cast<unsigned>(k.w[j >> 3] >> (8 * (j & 7))) & 0xffu;
      const uint64_t* e = tab + (static_cast<unsigned>(j) * 256u + b) * W;
      if constexpr (W == 1) {
        p.w[0] |= e[0];
      } else {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(e);
        p.w[0] |= v.x;
        p.w[1] |= v.y;
      }
    }
  }
  return p;
}

// Field [off, off+nb) of a packed word (nb <= 63).
template <int W>
__device__ __forceinline__ long long packed_field(const Key<W>& p, int off, int nb) {
  if (nb == 0) return 0;
  uint64_t v;
  if constexpr (W == 1) {
    v = p.w[0] >> off;
  } else {
    if (off >= 64) {
      v = p.w[1] >> (off - 64);
    } else if (off == 0) {
      v = p.w[0];
    } else {
      v = (p.w[0] >> off) | (p.w[1] << (64 - off));
    }
  }
  return static_cast<long long>(v & ((nb >= 64) ? ~0ull : ((1ull << nb) - 1ull)));
}

// Cooperative copy of `n_u64` words global -> shared.
__device__ __forceinline__ void copy_to_smem(uint64_t* dst, const uint64_t* __restrict__ src, int n_u64) {
  for (int i = threadIdx.x; i < n_u64; i += blockDim.x) dst[i] = __ldg(src + i);
}

// Partition id of element i for count ranges of near-equal size with the
// larger ranges first (format.py:136-140): sizes base+1 for l < extra.
__device__ __forceinline__ long long partition_of(long long i, long long base, long long extra) {
  const long long big = extra * (base + 1);
  if (i < big) return i / (base + 1);
  return extra + (i - big) / base;
}

}  // namespace alto
