// Experiment (round 2): the FT6D key transpose done entirely by the TMA engine.
//
// FasterTransformer's key layout is packet-major: [slab][u = D*e/16 packets][S positions][16 B]
// (NEXT-1). The wire is position-major: [slab][n positions][u][16 B]. A tile of
// TS positions x all U packets is loaded by ONE cp.async.bulk.tensor from a tensor map over the
// cache (dims: 16-B packet, position (stride 16 B), packet index (stride S*16), slab) into shared
// memory as [u][s][16 B], and stored by ONE cp.async.bulk.tensor through a tensor map over the
// wire whose dims are listed in the SAME order -- position with stride D*e, packet index with
// stride 16 B -- so the TMA engine performs the 16-byte transpose on the store; no thread touches
// a byte. Form "tma": that; form "tma_smem": TMA load, threads transpose in shared memory, one
// plain bulk store of the contiguous TS*256-B wire tile; form "ldg": the register transpose
// baseline (one thread = one position, 16 x 16-B loads, 8 x 32-B stores).
//
// Reports device us per pack of positions [0, N) of every slab and GB/s at 2R against the HBM peak,
// after checking every wire word against a direct index computation.
//
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -o tools/tma_ft6d_probe tools/tma_ft6d_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                           \
    }                                                                                    \
  } while (0)

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q));
  if (!f || q != cudaDriverEntryPointSuccess) {
    fprintf(stderr, "no cuTensorMapEncodeTiled\n");
    exit(1);
  }
  return (EncodeFn)f;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load4(const CUtensorMap* m, void* dst, uint64_t* bar, int c0, int c1, int c2,
                                          int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap* m, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_store4(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(m),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

constexpr int U = 16;  // packets of a D = 128 fp16 row

// Pure TMA: one elected thread per CTA runs an NST-deep load pipeline; each loaded tile is stored
// through the transposing wire map. Tiles: slab-major, TS positions each.
template <int TS, int NST, int MODE>
__global__ void __launch_bounds__(32) k_tma(const __grid_constant__ CUtensorMap src_map,
                                            const __grid_constant__ CUtensorMap dst_map, int n_slabs, int N) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[NST];
  if (threadIdx.x != 0) return;
  const int tiles_per_slab = (N + TS - 1) / TS;
  const int n_tiles = n_slabs * tiles_per_slab;
  for (int i = 0; i < NST; ++i) mbar_init(&bar[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int first = blockIdx.x, stride = gridDim.x;
  const int mine = first < n_tiles ? (n_tiles - first + stride - 1) / stride : 0;
  auto issue = [&](int j) {
    const int t = first + j * stride;
    const int slab = t / tiles_per_slab, s0 = (t % tiles_per_slab) * TS;
    uint8_t* buf = sm + (j % NST) * (TS * U * 16);
    mbar_expect(&bar[j % NST], TS * U * 16);
    if (MODE == 0)
      tma_load4(&src_map, buf, &bar[j % NST], 0, s0, 0, slab);
    else
      tma_load4(&src_map, buf, &bar[j % NST], 0, 0, s0, slab);
  };
  for (int j = 0; j < (NST < mine ? NST : mine); ++j) issue(j);
  for (int j = 0; j < mine; ++j) {
    const int t = first + j * stride;
    const int slab = t / tiles_per_slab, s0 = (t % tiles_per_slab) * TS;
    mbar_wait(&bar[j % NST], (j / NST) & 1);
    if (MODE == 0)
      tma_store4(&dst_map, sm + (j % NST) * (TS * U * 16), 0, s0, 0, slab);
    else
      tma_store3(&dst_map, sm + (j % NST) * (TS * U * 16), 0, s0, slab);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (j >= 1 && j - 1 + NST < mine) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // store j-1 has read its stage
      issue(j - 1 + NST);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Register transpose baseline: one thread = one (slab, position): 16 packet loads (a warp's 32
// positions of one packet = one 512-B segment), one 256-B row store.
__global__ void __launch_bounds__(256) k_ldg(const uint4* __restrict__ src, uint4* __restrict__ dst, int n_slabs,
                                             int S, int N) {
  const int64_t total = (int64_t)n_slabs * N;
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int64_t slab = i / N;
    const int s = (int)(i % N);
    uint4 v[U];
    const uint4* a = src + slab * U * S + s;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + (int64_t)u * S);
    uint4* d = dst + (slab * N + s) * U;
#pragma unroll
    for (int u = 0; u < U; ++u) d[u] = v[u];
  }
}

__device__ __forceinline__ void st_v8(void* p, const uint4& a, const uint4& b) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w),
               "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

// Hybrid: the TMA engine loads whole packet rows (box inner dim TS*16 B contiguous, U rows) into
// shared memory [u][s][16 B]; the CTA's threads then read two packets of one position from shared
// memory and store them as one 32-byte vector (a warp's lanes walk 32 positions of one packet pair:
// conflict-free 16-B shared reads, full 32-B sectors on the global side). Thread 0 keeps NST tile
// loads in flight; one TMA box per packet row (128-B aligned shared rows of TS*16 bytes).
template <int TS, int NST>
__global__ void __launch_bounds__(256) k_tma_hybrid(const __grid_constant__ CUtensorMap src_map, uint8_t* wire,
                                                    int n_slabs, int N) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[NST];
  constexpr int ROW = TS * 16;
  constexpr int STAGE = U * ROW;
  const int tiles_per_slab = (N + TS - 1) / TS;
  const int n_tiles = n_slabs * tiles_per_slab;
  const int first = blockIdx.x, stride = gridDim.x;
  const int mine = first < n_tiles ? (n_tiles - first + stride - 1) / stride : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int j) {
    const int t = first + j * stride;
    const int slab = t / tiles_per_slab, s0 = (t % tiles_per_slab) * TS;
    uint8_t* buf = sm + (j % NST) * STAGE;
    mbar_expect(&bar[j % NST], TS * U * 16);
    for (int u = 0; u < U; ++u)   // one 2-D box per packet row: (TS*4 words, 1 row)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              smem_u32(buf + u * ROW)),
          "l"(&src_map), "r"(s0 * 4), "r"(u), "r"(slab), "r"(smem_u32(&bar[j % NST]))
          : "memory");
  };
  if (threadIdx.x == 0)
    for (int j = 0; j < (NST < mine ? NST : mine); ++j) issue(j);
  for (int j = 0; j < mine; ++j) {
    const int t = first + j * stride;
    const int slab = t / tiles_per_slab, s0 = (t % tiles_per_slab) * TS;
    const int ns = min(TS, N - s0);
    mbar_wait(&bar[j % NST], (j / NST) & 1);
    const uint8_t* buf = sm + (j % NST) * STAGE;
    uint8_t* out = wire + ((size_t)slab * N + s0) * (U * 16);
    for (int i = threadIdx.x; i < TS * (U / 2); i += 256) {
      const int s = i % TS, pr = i / TS;
      if (s >= ns) continue;
      const uint4 a = *(const uint4*)(buf + (2 * pr) * ROW + s * 16);
      const uint4 b = *(const uint4*)(buf + (2 * pr + 1) * ROW + s * 16);
      st_v8(out + (size_t)s * (U * 16) + pr * 32, a, b);
    }
    __syncthreads();   // every thread is done reading this stage
    if (threadIdx.x == 0 && j + NST < mine) issue(j + NST);
  }
}

// Register transpose as the library does it (PK = 16): 16 x 16-B loads of one position, 8 x 32-B stores.
__global__ void __launch_bounds__(256) k_ldg32(const uint4* __restrict__ src, uint8_t* __restrict__ dst, int n_slabs,
                                               int S, int N) {
  const int64_t total = (int64_t)n_slabs * N;
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int64_t slab = i / N;
    const int s = (int)(i % N);
    uint4 v[U];
    const uint4* a = src + slab * U * S + s;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + (int64_t)u * S);
    uint8_t* d = dst + (slab * N + s) * U * 16;
#pragma unroll
    for (int u = 0; u < U; u += 2) st_v8(d + u * 16, v[u], v[u + 1]);
  }
}

__global__ void k_fill(uint32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    p[i] = (uint32_t)(i * 2654435761ull ^ (i >> 7));
}
// wire word w of (slab, s, u, c) must equal cache word of (slab, u, s, c)
__global__ void k_check(const uint32_t* cache, const uint32_t* wire, int n_slabs, int S, int N,
                        unsigned long long* bad) {
  const int64_t total = (int64_t)n_slabs * N * U * 4;
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int c = i % 4;
    const int u = (i / 4) % U;
    const int s = (i / (4 * U)) % N;
    const int64_t slab = i / (4 * U * (int64_t)N);
    const uint32_t want = cache[((slab * U + u) * S + s) * 4 + c];
    if (wire[i] != want) atomicAdd(bad, 1ull);
  }
}

int main(int argc, char** argv) {
  const int L = 1, B = 8, H = 40, S = 2048, N = argc > 1 ? atoi(argv[1]) : 1000;
  const int n_layers_ring = 8;  // cycle through 8 layers so the source is not L2-resident
  const int n_slabs = L * B * H;
  const size_t slab_bytes = (size_t)U * S * 16;
  const size_t cache_bytes = slab_bytes * n_slabs * n_layers_ring;
  const size_t wire_bytes = (size_t)n_slabs * N * U * 16;
  uint8_t *cache, *wire;
  unsigned long long* bad;
  CK(cudaMalloc(&cache, cache_bytes));
  CK(cudaMalloc(&wire, wire_bytes * 2));
  CK(cudaMalloc(&bad, 8));
  k_fill<<<4096, 256>>>((uint32_t*)cache, cache_bytes / 4);
  CK(cudaDeviceSynchronize());
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  EncodeFn enc = encode_fn();

  // maps per layer of the ring: [0] = MODE 0 (plain load, transposing store), [1] = MODE 1
  const int TS = 64;
  std::vector<CUtensorMap> smaps[3];
  CUtensorMap dmap[2][2];
  auto check = [](CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) {
      printf("{\"error\": \"%s encode %d\"}\n", what, (int)r);
      fflush(stdout);
      return false;
    }
    return true;
  };
  bool ok_mode[3] = {true, true, true};
  cuuint32_t es[4] = {1, 1, 1, 1};
  for (int l = 0; l < n_layers_ring; ++l) {
    void* base = cache + (size_t)l * slab_bytes * n_slabs;
    CUtensorMap m0, m1;
    cuuint64_t gd0[4] = {4, (cuuint64_t)S, (cuuint64_t)U, (cuuint64_t)n_slabs};
    cuuint64_t gs0[3] = {16, (cuuint64_t)S * 16, (cuuint64_t)U * S * 16};
    cuuint32_t box0[4] = {4, TS, U, 1};
    ok_mode[0] &= check(enc(&m0, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, base, gd0, gs0, box0, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                        "mode0 source");
    cuuint64_t gd1[4] = {4, (cuuint64_t)U, (cuuint64_t)S, (cuuint64_t)n_slabs};
    cuuint64_t gs1[3] = {(cuuint64_t)S * 16, 16, (cuuint64_t)U * S * 16};  // packet stride S*16, position 16
    cuuint32_t box1[4] = {4, U, TS, 1};
    ok_mode[1] &= check(enc(&m1, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, base, gd1, gs1, box1, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                        "mode1 source (transposing)");
    CUtensorMap m2;
    cuuint64_t gd2[3] = {(cuuint64_t)S * 4, (cuuint64_t)U, (cuuint64_t)n_slabs};
    cuuint64_t gs2[2] = {(cuuint64_t)S * 16, (cuuint64_t)U * S * 16};
    cuuint32_t box2[3] = {TS * 4, 1, 1};
    ok_mode[2] &= check(enc(&m2, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, base, gd2, gs2, box2, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                        "hybrid source rows");
    smaps[2].push_back(m2);
    smaps[0].push_back(m0);
    smaps[1].push_back(m1);
  }
  for (int w = 0; w < 2; ++w) {
    cuuint64_t gd0[4] = {4, (cuuint64_t)N, (cuuint64_t)U, (cuuint64_t)n_slabs};
    cuuint64_t gs0[3] = {(cuuint64_t)U * 16, 16, (cuuint64_t)N * U * 16};  // position stride 256, packet stride 16
    cuuint32_t box0[4] = {4, TS, U, 1};
    ok_mode[0] &= check(enc(&dmap[0][w], CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, wire + w * wire_bytes, gd0, gs0, box0, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                        "mode0 wire (transposing)");
    cuuint64_t gd1[3] = {(cuuint64_t)U * 4, (cuuint64_t)N, (cuuint64_t)n_slabs};
    cuuint64_t gs1[2] = {(cuuint64_t)U * 16, (cuuint64_t)N * U * 16};
    cuuint32_t box1[3] = {(cuuint32_t)U * 4, TS, 1};
    ok_mode[1] &= check(enc(&dmap[1][w], CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, wire + w * wire_bytes, gd1, gs1, box1, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                        "mode1 wire");
  }
  const int NST = 4;
  const int smem = NST * TS * U * 16;
  CK(cudaFuncSetAttribute(k_tma<TS, NST, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_tma<TS, NST, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int smem_h = NST * U * TS * 16;
  CK(cudaFuncSetAttribute(k_tma_hybrid<TS, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_h));
  const int tiles = n_slabs * ((N + TS - 1) / TS);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const double bytes2r = 2.0 * wire_bytes;
  const char* names[5] = {"tma_store_transpose", "tma_load_transpose", "ldg_regs16", "tma_rows_smem_stg32",
                          "ldg_regs_stg32"};
  for (int form = 0; form < 5; ++form) {
    if (form < 2 && !ok_mode[form]) continue;
    if (form == 3 && !ok_mode[2]) continue;
    for (int per_sm : {1, 2, 3, 4, 6, 8}) {
      if ((form == 2 || form == 4) && per_sm != 8) continue;
      const int grid = (form < 2 || form == 3) ? std::min(tiles, nsm * per_sm) : nsm * 8;
      auto run = [&](int it) {
        const int l = it % n_layers_ring;
        if (form == 0)
          k_tma<TS, NST, 0><<<grid, 32, smem>>>(smaps[0][l], dmap[0][it & 1], n_slabs, N);
        else if (form == 1)
          k_tma<TS, NST, 1><<<grid, 32, smem>>>(smaps[1][l], dmap[1][it & 1], n_slabs, N);
        else if (form == 3)
          k_tma_hybrid<TS, NST><<<grid, 256, smem_h>>>(smaps[2][l], wire + (it & 1) * wire_bytes, n_slabs, N);
        else if (form == 4)
          k_ldg32<<<grid, 256>>>((const uint4*)(cache + (size_t)l * slab_bytes * n_slabs),
                                 wire + (it & 1) * wire_bytes, n_slabs, S, N);
        else
          k_ldg<<<grid, 256>>>((const uint4*)(cache + (size_t)l * slab_bytes * n_slabs),
                               (uint4*)(wire + (it & 1) * wire_bytes), n_slabs, S, N);
      };
      // parity: call it0 = 3 packs ring layer 3 into wire 1 (wire pre-filled with 0xff)
      const int it0 = 3;
      const int l0 = it0 % n_layers_ring, w0 = it0 & 1;
      CK(cudaMemset(wire + w0 * wire_bytes, 0xff, wire_bytes));
      run(it0);
      CK(cudaDeviceSynchronize());
      CK(cudaMemset(bad, 0, 8));
      k_check<<<4096, 256>>>((const uint32_t*)(cache + (size_t)l0 * slab_bytes * n_slabs),
                             (const uint32_t*)(wire + w0 * wire_bytes), n_slabs, S, N, bad);
      unsigned long long nbad = 0;
      CK(cudaMemcpy(&nbad, bad, 8, cudaMemcpyDeviceToHost));
      for (int i = 0; i < 5; ++i) run(i);
      CK(cudaDeviceSynchronize());
      std::vector<float> ts;
      for (int rep = 0; rep < 7; ++rep) {
        CK(cudaEventRecord(a));
        const int n = 40;
        for (int i = 0; i < n; ++i) run(rep * n + i);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        ts.push_back(ms * 1000.f / n);
      }
      std::sort(ts.begin(), ts.end());
      const double us = ts[3];
      printf("{\"form\": \"%s\", \"N\": %d, \"TS\": %d, \"NST\": %d, \"grid\": %d, \"bytes\": %zu, \"us\": %.2f, "
             "\"gbs_2R\": %.1f, \"frac_hbm\": %.3f, \"mismatches\": %llu}\n",
             names[form], N, TS, NST, grid, wire_bytes, us, bytes2r / us / 1e3, bytes2r / us / 1e3 / 6544.0, nbad);
      fflush(stdout);
    }
  }
  return 0;
}
