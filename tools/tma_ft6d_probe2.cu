// Experiment (round 2, follow-up of tools/tma_ft6d_probe.cu): the FT6D key transpose with the TMA
// engine on the packet-major side only, against the register transpose, in BOTH directions, under
// the library's measurement conditions (C2 prompt layer K half: 8 x 40 slabs x N positions, source
// layers cycled over a 12-layer ring, one wire buffer, median of 7 x 20 launches).
//
//   pack   (FT6D -> wire): TMA loads whole packet rows (one 2-D box of TS*16 B per packet) into
//          shared memory [u][s]; threads read two packets of one position and store 32 B.
//   unpack (wire -> FT6D): threads load 32 B (two packets of one position) and write them to
//          shared memory [u][s]; after a proxy fence + barrier thread 0 stores each packet row with
//          one TMA box (clipped at the region's end by the map's extent: bytes past the region are
//          never written).
//   regs:  one thread = one position, 16 x 16-B packet accesses on the FT6D side, 8 x 32-B on the wire.
//
// Every output word is checked (pack: wire vs cache; unpack: region words vs wire, and the words
// just past the region untouched).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -o tools/tma_ft6d_probe2 tools/tma_ft6d_probe2.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

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

constexpr int U = 16;

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
__device__ __forceinline__ void st_v8(void* p, const uint4& a, const uint4& b) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w),
               "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}
__device__ __forceinline__ void ld_v8(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 a;
  asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w)
               : "l"(p));
  return a;
}

// pack: TMA rows in, threads out
template <int TS, int NST>
__global__ void __launch_bounds__(256) k_pack_hybrid(const __grid_constant__ CUtensorMap rows, uint8_t* wire,
                                                     int n_slabs, int N) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[NST];
  constexpr int STAGE = U * TS * 16;
  const int tps = (N + TS - 1) / TS, n_tiles = n_slabs * tps;
  const int first = blockIdx.x, stride = gridDim.x;
  const int mine = first < n_tiles ? (n_tiles - first + stride - 1) / stride : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int j) {
    const int t = first + j * stride, slab = t / tps, s0 = (t % tps) * TS;
    uint8_t* buf = sm + (j % NST) * STAGE;
    mbar_expect(&bar[j % NST], STAGE);
    for (int u = 0; u < U; ++u)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              smem_u32(buf + u * TS * 16)),
          "l"(&rows), "r"(s0 * 4), "r"(u), "r"(slab), "r"(smem_u32(&bar[j % NST]))
          : "memory");
  };
  if (threadIdx.x == 0)
    for (int j = 0; j < (NST < mine ? NST : mine); ++j) issue(j);
  for (int j = 0; j < mine; ++j) {
    const int t = first + j * stride, slab = t / tps, s0 = (t % tps) * TS;
    const int ns = min(TS, N - s0);
    mbar_wait(&bar[j % NST], (j / NST) & 1);
    const uint8_t* buf = sm + (j % NST) * STAGE;
    uint8_t* out = wire + ((size_t)slab * N + s0) * (U * 16);
#pragma unroll
    for (int k = 0; k < TS * (U / 2) / 256; ++k) {
      const int i = k * 256 + threadIdx.x, s = i % TS, pr = i / TS;
      if (s < ns) {
        const uint4 a = *(const uint4*)(buf + (2 * pr) * TS * 16 + s * 16);
        const uint4 b = *(const uint4*)(buf + (2 * pr + 1) * TS * 16 + s * 16);
        st_v8(out + (size_t)s * (U * 16) + pr * 32, a, b);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && j + NST < mine) issue(j + NST);
  }
}

// unpack: threads in, TMA rows out
template <int TS, int NST>
__global__ void __launch_bounds__(256) k_unpack_hybrid(const uint8_t* wire, const __grid_constant__ CUtensorMap rows,
                                                       int n_slabs, int N) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int STAGE = U * TS * 16;
  const int tps = (N + TS - 1) / TS, n_tiles = n_slabs * tps;
  int j = 0;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++j) {
    const int slab = t / tps, s0 = (t % tps) * TS, ns = min(TS, N - s0);
    uint8_t* buf = sm + (j % NST) * STAGE;
    if (j >= NST) {   // the stores that read this stage NST tiles ago are done reading it
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NST - 1) : "memory");
      __syncthreads();
    }
    const uint8_t* in = wire + ((size_t)slab * N + s0) * (U * 16);
    constexpr int IT = TS * (U / 2) / 256;
    uint4 a[IT], b[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int i = k * 256 + threadIdx.x, s = i % TS, pr = i / TS;
      if (s < ns) ld_v8(in + (size_t)s * (U * 16) + pr * 32, a[k], b[k]);
    }
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int i = k * 256 + threadIdx.x, s = i % TS, pr = i / TS;
      if (s < ns) {
        *(uint4*)(buf + (2 * pr) * TS * 16 + s * 16) = a[k];
        *(uint4*)(buf + (2 * pr + 1) * TS * 16 + s * 16) = b[k];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int u = 0; u < U; ++u)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                         &rows),
                     "r"(smem_u32(buf + u * TS * 16)), "r"(s0 * 4), "r"(u), "r"(slab)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// register forms (the library's PK = 16 item): one thread = one position
__global__ void __launch_bounds__(256) k_pack_regs(const uint8_t* __restrict__ cache, uint8_t* __restrict__ wire,
                                                   int n_slabs, int S, int N) {
  const int64_t total = (int64_t)n_slabs * N;
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int64_t slab = i / N;
    const int s = (int)(i % N);
    uint4 v[U];
    const uint8_t* a = cache + (slab * U * S + s) * 16;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_v4(a + (int64_t)u * S * 16);
    uint8_t* d = wire + (slab * N + s) * U * 16;
#pragma unroll
    for (int u = 0; u < U; u += 2) st_v8(d + u * 16, v[u], v[u + 1]);
  }
}
__global__ void __launch_bounds__(256) k_unpack_regs(const uint8_t* __restrict__ wire, uint8_t* __restrict__ cache,
                                                     int n_slabs, int S, int N) {
  const int64_t total = (int64_t)n_slabs * N;
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int64_t slab = i / N;
    const int s = (int)(i % N);
    uint4 v[U];
    const uint8_t* a = wire + (slab * N + s) * U * 16;
#pragma unroll
    for (int u = 0; u < U; u += 2) ld_v8(a + u * 16, v[u], v[u + 1]);
    uint8_t* d = cache + (slab * U * S + s) * 16;
#pragma unroll
    for (int u = 0; u < U; ++u) *(uint4*)(d + (int64_t)u * S * 16) = v[u];
  }
}

__global__ void k_fill(uint32_t* p, int64_t n, uint32_t salt) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    p[i] = (uint32_t)(i * 2654435761ull ^ (i >> 7) ^ salt);
}
// every (slab, s < N, u, c) word: wire == cache; and (DIR 1) cache words at s in [N, N+64) keep the sentinel
__global__ void k_check(const uint32_t* cache, const uint32_t* wire, int n_slabs, int S, int N, int check_tail,
                        uint32_t sentinel, unsigned long long* bad) {
  const int64_t total = (int64_t)n_slabs * N * U * 4;
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int c = i % 4, u = (i / 4) % U, s = (i / (4 * U)) % N;
    const int64_t slab = i / (4 * U * (int64_t)N);
    if (wire[i] != cache[((slab * U + u) * S + s) * 4 + c]) atomicAdd(bad, 1ull);
    if (check_tail && s < 64 && N + s < S && cache[((slab * U + u) * S + N + s) * 4 + c] != sentinel)
      atomicAdd(bad, 1ull);
  }
}

static EncodeFn g_enc;
static CUtensorMap rows_map(void* base, int n_slabs, int S, int extent, int TS) {
  CUtensorMap m;
  cuuint64_t gd[3] = {(cuuint64_t)extent * 4, (cuuint64_t)U, (cuuint64_t)n_slabs};
  cuuint64_t gs[2] = {(cuuint64_t)S * 16, (cuuint64_t)U * S * 16};
  cuuint32_t box[3] = {(cuuint32_t)TS * 4, 1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, base, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("{\"error\": \"encode %d\"}\n", (int)r);
    exit(1);
  }
  return m;
}

int main(int argc, char** argv) {
  const int B = 8, H = 40, S = 2048, N = argc > 1 ? atoi(argv[1]) : 1000;
  const int RING = 12, n_slabs = B * H;
  const size_t layer_bytes = (size_t)n_slabs * U * S * 16;
  const size_t wire_bytes = (size_t)n_slabs * N * U * 16;
  uint8_t *cache, *wire;
  unsigned long long* bad;
  CK(cudaMalloc(&cache, layer_bytes * RING));
  CK(cudaMalloc(&wire, wire_bytes));
  CK(cudaMalloc(&bad, 8));
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q));
  g_enc = (EncodeFn)f;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double b2r = 2.0 * wire_bytes;

  struct Form {
    const char* name;
    int dir;   // 0 pack, 1 unpack
    int ts, nst, per_sm;
  };
  std::vector<Form> forms;
  for (int dir = 0; dir < 2; ++dir) {
    forms.push_back({"regs", dir, 0, 0, 8});
    for (int ts : {32, 64})
      for (int nst : {2, 3, 4})
        for (int per_sm : {1, 2, 3}) forms.push_back({"tma_hybrid", dir, ts, nst, per_sm});
  }
  std::vector<CUtensorMap> maps_full(RING), maps_N(RING);
  for (const Form& fm : forms) {
    const int TS = fm.ts ? fm.ts : 64;
    for (int l = 0; l < RING; ++l) {
      maps_full[l] = rows_map(cache + l * layer_bytes, n_slabs, S, S, TS);
      maps_N[l] = rows_map(cache + l * layer_bytes, n_slabs, S, N, TS);
    }
    const int smem = fm.nst * U * TS * 16;
    const int tiles = n_slabs * ((N + TS - 1) / TS);
    const int grid = fm.ts ? std::min(tiles, nsm * fm.per_sm) : nsm * fm.per_sm;
#define SETSM(K) CK(cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))
    if (fm.ts == 32 && fm.nst == 2) { SETSM((k_pack_hybrid<32, 2>)); SETSM((k_unpack_hybrid<32, 2>)); }
    if (fm.ts == 32 && fm.nst == 3) { SETSM((k_pack_hybrid<32, 3>)); SETSM((k_unpack_hybrid<32, 3>)); }
    if (fm.ts == 32 && fm.nst == 4) { SETSM((k_pack_hybrid<32, 4>)); SETSM((k_unpack_hybrid<32, 4>)); }
    if (fm.ts == 64 && fm.nst == 2) { SETSM((k_pack_hybrid<64, 2>)); SETSM((k_unpack_hybrid<64, 2>)); }
    if (fm.ts == 64 && fm.nst == 3) { SETSM((k_pack_hybrid<64, 3>)); SETSM((k_unpack_hybrid<64, 3>)); }
    if (fm.ts == 64 && fm.nst == 4) { SETSM((k_pack_hybrid<64, 4>)); SETSM((k_unpack_hybrid<64, 4>)); }
    auto run = [&](int it) {
      const int l = it % RING;
      uint8_t* lc = cache + l * layer_bytes;
#define HY(T, NS)                                                                                   \
  if (fm.ts == T && fm.nst == NS) {                                                                 \
    if (fm.dir == 0)                                                                                \
      k_pack_hybrid<T, NS><<<grid, 256, smem>>>(maps_full[l], wire, n_slabs, N);                    \
    else                                                                                            \
      k_unpack_hybrid<T, NS><<<grid, 256, smem>>>(wire, maps_N[l], n_slabs, N);                     \
  }
      if (!fm.ts) {
        if (fm.dir == 0)
          k_pack_regs<<<grid, 256>>>(lc, wire, n_slabs, S, N);
        else
          k_unpack_regs<<<grid, 256>>>(wire, lc, n_slabs, S, N);
      }
      HY(32, 2) HY(32, 3) HY(32, 4) HY(64, 2) HY(64, 3) HY(64, 4)
    };
    // parity on ring layer 5
    const uint32_t sentinel = 0xDEADBEEFu;
    if (fm.dir == 0) {
      k_fill<<<4096, 256>>>((uint32_t*)cache, layer_bytes * RING / 4, 0);
      CK(cudaMemset(wire, 0xff, wire_bytes));
    } else {
      k_fill<<<4096, 256>>>((uint32_t*)wire, wire_bytes / 4, 77);
      std::vector<uint32_t> h(layer_bytes / 4, sentinel);
      CK(cudaMemcpy(cache + 5 * layer_bytes, h.data(), layer_bytes, cudaMemcpyHostToDevice));
    }
    run(5);
    CK(cudaDeviceSynchronize());
    CK(cudaMemset(bad, 0, 8));
    k_check<<<4096, 256>>>((const uint32_t*)(cache + 5 * layer_bytes), (const uint32_t*)wire, n_slabs, S, N,
                           fm.dir, sentinel, bad);
    unsigned long long nbad = 0;
    CK(cudaMemcpy(&nbad, bad, 8, cudaMemcpyDeviceToHost));
    std::vector<float> ts;
    for (int rep = 0; rep < 7; ++rep) {
      run(rep);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      for (int i = 0; i < 20; ++i) run(rep * 20 + i + 1);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ts.push_back(ms * 1000.f / 20);
    }
    std::sort(ts.begin(), ts.end());
    printf("{\"dir\": \"%s\", \"form\": \"%s\", \"N\": %d, \"TS\": %d, \"NST\": %d, \"grid\": %d, \"us\": %.2f, "
           "\"frac_2R\": %.3f, \"mismatches\": %llu}\n",
           fm.dir ? "unpack" : "pack", fm.name, N, fm.ts, fm.nst, grid, ts[3], b2r / ts[3] / 1e3 / 6544.0, nbad);
    fflush(stdout);
  }
  return 0;
}
