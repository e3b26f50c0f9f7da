// psg_project_tc.cu — K1, the projection keys[i][k] = <U_k, X_i>, as a
// TMA-fed tcgen05 GEMM (BASELINE.json north_star item 1; the reference's
// counterpart is the reference-distance table of build_reference_set,
// refscan.cpp:30-65, whose role the projection keys take over).
//
// D = X (n x d, FP32 rows) . U^T (d x 16): M = 128 rows per tile, N = 16 (the
// nk <= 8 directions zero-padded), K = d in 32-float chunks.  X is split
// exactly into two TF32 terms, x = hi + lo (hi = x with its 13 low mantissa
// bits cleared, lo = x - hi), and both are multiplied: near-FP32 keys.
//
//   warp 0 (one thread)  TMA producer: one 128-row x 32-float box (16 KB, 128 B
//                        swizzle) per smem stage, kTcStages in flight; the
//                        tail tile's OOB rows are zero-filled
//   warps 4-7, 12-15     split (two groups, alternate chunks): lane = row; each thread reads its row's 32
//                        floats of a stage (conflict-free through the swizzle),
//                        frees the stage, and writes hi | lo to a TMEM slot
//                        (tcgen05.st 32x32b, 64 columns per slot, kTcSlots)
//   warp 1 (one thread)  MMA issuer: per slot 2 x 4 tcgen05.mma.kind::tf32
//                        (A = hi / lo from TMEM, B = U from smem, K = 8 each)
//                        into two TMEM accumulator chains (hi, lo: 2 x 16
//                        columns, double buffered across tiles, summed by the
//                        epilogue); tcgen05.commit frees the slot
//                        and, after a tile's last chunk, hands it to the epilogue
//   warps 8-11           epilogue: tcgen05.ld 32x32b (lane = row) -> nk keys
//                        per row, 32 B coalesced stores
//   warp 2               TMEM allocation / release (all 512 columns)
//
// Persistent: one CTA per SM walks tiles blockIdx.x, +gridDim.x, ...  Shared
// memory carries only the TMA stream (read once by the split warps); the
// operand traffic of the MMAs is TMEM's.
//
// Precision: U is rounded to TF32 when the directions are made
// (psg_points.cu), so it is an exact operand; hi is exact TF32, lo enters as
// TF32 (<= 2^-10 |lo| <= 2^-20 |x| lost), products are exact in FP32 and the
// accumulation is FP32 in the tensor core.  key_gamma/key_abs
// (psg_internal.cuh) charge this, with margin, as the key error E of the
// filter budget — the "explicit rounding slack on the filter bound"; every
// decision is still taken by the FP64 recheck, so answers stay exact, and
// tests/test_gpu_keys.py checks the charged E against FP64 projections.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>

#include "psg_cpp.cuh"
#include "psg_tc.cuh"

namespace psg {
namespace {

using namespace tc;

constexpr int kTcM = 128;         // rows per tile (UMMA M)
constexpr int kTcN = 16;          // UMMA N: directions padded to 16
constexpr int kTcKChunk = 32;     // floats per 128 B swizzle row = one pipeline stage
constexpr int kTcStages = 8;      // smem stages: 8 x 16 KB in flight per SM
constexpr int kTcSlots = 7;       // TMEM A slots (64 columns: hi | lo) after the accumulators
constexpr uint32_t kStageBytes = kTcM * kTcKChunk * 4;  // 16 KB
constexpr uint32_t kBChunkBytes = kTcN * 128;            // 2 KB: 16 rows x 128 B
constexpr int kTcThreads = 512;
constexpr uint32_t kTmemCols = 512;  // [0, 64) 2 x (hi, lo) accumulators, [64, 64 + 64 kTcSlots) A slots
constexpr uint32_t kSlotBase = 64;

constexpr uint32_t kIdesc = idesc_tf32(kTcM, kTcN);  // D F32, A/B TF32, K-major, M = 128, N = 16

template <int D>
struct UTc {
  float u[8][D];  // rows >= nk are zero
};

template <int NK, int D>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_project_tc(const __grid_constant__ CUtensorMap xmap, uint32_t n, const __grid_constant__ UTc<D> U,
                 float* __restrict__ keys, unsigned* __restrict__ norm2_bits, unsigned set_norm2_bits, CellCount cc) {
  constexpr int NC = D / kTcKChunk;  // K chunks (stages) per tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared pointer
  uint8_t* sa = smem;                             // kTcStages x 16 KB (A stages)
  uint8_t* sb = smem + kTcStages * kStageBytes;   // NC x 2 KB (B = U, SW128 K-major)
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + NC * kBChunkBytes);  // TMA -> split   (tx)
  uint64_t* sfree = full + kTcStages;                                     // split -> TMA   (4 warps)
  uint64_t* tready = sfree + kTcStages;                                   // split -> MMA   (4 warps)
  uint64_t* tslot = tready + kTcSlots;                                    // MMA -> split   (commit)
  uint64_t* tfull = tslot + kTcSlots;                                     // MMA -> epilogue (commit)
  uint64_t* tempty = tfull + 2;                                           // epilogue -> MMA (4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // B operand once per CTA: row r (direction), float kk of chunk c lands in
  // 16 B unit (kk/4) ^ (r%8) of the row's 128 B (the 128 B swizzle pattern)
  for (int i = threadIdx.x; i < kTcN * D; i += kTcThreads) {
    const int r = i / D, k = i % D, c = k / kTcKChunk, kk = k % kTcKChunk;
    const float v = r < NK ? U.u[r][k] : 0.f;
    const uint32_t off = c * kBChunkBytes + r * 128 + ((((kk >> 2) ^ (r & 7)) & 7) << 4) + (kk & 3) * 4;
    *reinterpret_cast<float*>(sb + off) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> visible to the MMA (async proxy)
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(sfree + s, 4);
    }
    for (int s = 0; s < kTcSlots; ++s) {
      mbar_init(tready + s, 4);
      mbar_init(tslot + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x == 0) atomicMax(norm2_bits, set_norm2_bits);  // the set's row norms (psg_pointset::norm2max)
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // PDL: the set-up above (B operand, barriers, TMEM) overlaps the
  // predecessor's tail.  When the epilogue counts cells (cc.gp) the predecessor
  // is k_presample, which started after everything before it had completed and
  // writes only what the epilogue reads (GridParams, the box, the big-cell
  // counters): the TMA producer and the MMA warp then start on X at once and
  // only the epilogue warps wait, so the mainloop fills the TMEM slots and the
  // shared-memory ring while the sample is still being reduced.
  const bool early = cc.gp != nullptr;
  if (!early) {
    pdl_wait();
    pdl_trigger();
  }
  const uint32_t tmem = *tmem_slot;
  const uint32_t ntiles = (n + kTcM - 1) / kTcM;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int c = 0; c < NC; ++c) {
          mbar_wait(sfree + stage, phase ^ 1);
          mbar_arrive_expect_tx(full + stage, kStageBytes);
          tma_load_2d(sa + stage * kStageBytes, &xmap, full + stage, c * kTcKChunk, static_cast<int>(t * kTcM));
          if (++stage == kTcStages) {
            stage = 0;
            phase ^= 1;
          }
        }
    }
  } else if ((warp >= 4 && warp < 8) || warp >= 12) {
    // split: two groups of four warps take alternate chunks; warp w owns rows /
    // TMEM lanes 32 (w % 4) .. 32 (w % 4) + 31 (the tcgen05 lane-quarter rule)
    const uint32_t e = warp & 3, grp = warp >= 12, r = 32 * e + lane;
    const uint32_t lane_addr = tmem + ((32u * e) << 16) + kSlotBase;
    const uint32_t nchunks = (ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0) * NC;
    for (uint32_t j = grp; j < nchunks; j += 2) {
      const uint32_t stage = j % kTcStages, phase = (j / kTcStages) & 1;
      const uint32_t slot = j % kTcSlots, sphase = (j / kTcSlots) & 1;
      mbar_wait(full + stage, phase);
      const uint8_t* rowp = sa + stage * kStageBytes + r * 128;
      uint32_t hi[32], lo[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(rowp + ((q ^ (r & 7)) << 4));
        const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const uint32_t h = __float_as_uint(x[w]) & ~0x1fffu;
          hi[4 * q + w] = h;
          lo[4 * q + w] = __float_as_uint(x[w] - __uint_as_float(h));  // exact
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(sfree + stage);  // the TMA may refill this stage
      mbar_wait(tslot + slot, sphase ^ 1);        // the MMAs have consumed this slot's previous chunk
      tc_fence_after();
      tmem_st32(lane_addr + slot * 64, hi);
      tmem_st32(lane_addr + slot * 64 + 32, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tready + slot);
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp runs the loop (addresses stay in uniform
    // registers), one elected lane issues the MMAs and their commits
    uint32_t slot = 0, sphase = 0, it = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const uint32_t acc = it & 1, aphase = (it >> 1) & 1;
      mbar_wait(tempty + acc, aphase ^ 1);  // the epilogue has drained this accumulator
      tc_fence_after();
      const uint32_t dcol = tmem + acc * 2 * kTcN;  // two chains of 16 columns
      for (int c = 0; c < NC; ++c) {
        mbar_wait(tready + slot, sphase);  // hi | lo of this chunk are in TMEM
        tc_fence_after();
        const uint32_t a = tmem + kSlotBase + slot * 64;
        const uint64_t bd = sw128_desc(smem_u32(sb + c * kBChunkBytes));
        // hi products accumulate in chain 0, lo products in chain 1 (adjacent
        // MMAs are independent, so the tensor pipe overlaps them)
        static_assert(kTcKChunk == 32 && kTcN == 16, "umma_tf32_ts_chunk32 layout");
        if (elect_one()) {
          umma_tf32_ts_chunk32(dcol, a, bd, kIdesc, c != 0);
          umma_commit(tslot + slot);  // slot reusable once these MMAs have read it
        }
        __syncwarp();
        if (++slot == kTcSlots) {
          slot = 0;
          sphase ^= 1;
        }
      }
      if (elect_one()) umma_commit(tfull + acc);  // accumulator complete
      __syncwarp();
    }
  } else if (warp >= 8) {  // epilogue: warp (8 + e) owns TMEM lanes 32e .. 32e+31
    const uint32_t e = warp - 8;
    uint32_t it = 0;
    if (early) {
      pdl_wait();
      pdl_trigger();
    }
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const uint32_t acc = it & 1, aphase = (it >> 1) & 1;
      mbar_wait(tfull + acc, aphase);
      tc_fence_after();
      uint32_t r[8], r2[8];
      const uint32_t taddr = tmem + ((32u * e) << 16) + acc * 2 * kTcN;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(taddr));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=r"(r2[0]), "=r"(r2[1]), "=r"(r2[2]), "=r"(r2[3]), "=r"(r2[4]), "=r"(r2[5]), "=r"(r2[6]),
                     "=r"(r2[7])
                   : "r"(taddr + kTcN));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(r2[k]));  // hi + lo
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      const uint32_t row = t * kTcM + 32 * e + lane;
      if (row < n) {
        float4* out = reinterpret_cast<float4*>(keys + static_cast<size_t>(row) * NK);
        out[0] = make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]), __uint_as_float(r[3]));
        if constexpr (NK == 8)
          out[1] =
              make_float4(__uint_as_float(r[4]), __uint_as_float(r[5]), __uint_as_float(r[6]), __uint_as_float(r[7]));
        if (cc.gp) {  // the counting build's first step, on keys still in registers
          float k[NK];
#pragma unroll
          for (int q = 0; q < NK; ++q) k[q] = __uint_as_float(r[q]);
          count_cell<NK>(k, row, cc);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    PSG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw std::runtime_error("pairscan_b200: cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

template <int NK, int D>
void launch(const psg_pointset& ps, const Directions& dir, float* keys, unsigned* nb, cudaStream_t s,
            const CellCount& cc) {
  const uint32_t n = static_cast<uint32_t>(ps.n);
  if (n == 0) return;
  CUtensorMap map;
  const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(n)};
  const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(D) * sizeof(float)};
  const cuuint32_t box[2] = {kTcKChunk, kTcM};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ps.X), gdim, gstride, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("pairscan_b200: cuTensorMapEncodeTiled failed");
  UTc<D> u{};
  for (int k = 0; k < NK; ++k)
    for (int t = 0; t < D; ++t) u.u[k][t] = dir.U[static_cast<size_t>(k) * D + t];
  constexpr size_t kSmem = 1024 + kTcStages * kStageBytes + (D / kTcKChunk) * kBChunkBytes + 512;
  set_max_dynamic_smem(reinterpret_cast<const void*>(k_project_tc<NK, D>), kSmem);
  unsigned nbits;
  std::memcpy(&nbits, &ps.norm2max, 4);
  const uint32_t ntiles = (n + kTcM - 1) / kTcM;
  const int grid = static_cast<int>(std::min<uint32_t>(ntiles, static_cast<uint32_t>(ctx().sm_count)));
  launch_pdl(k_project_tc<NK, D>, grid, kTcThreads, kSmem, s, map, n, u, keys, nb, nbits, cc);
  PSG_LAUNCHED();
}

}  // namespace

void project_tc(const psg_pointset& ps, const Directions& dir, float* keys, unsigned* norm2_bits, cudaStream_t s,
                const CellCount& cc) {
  switch (dir.nk * 1000 + ps.d) {
    case 4032: launch<4, 32>(ps, dir, keys, norm2_bits, s, cc); break;
    case 4064: launch<4, 64>(ps, dir, keys, norm2_bits, s, cc); break;
    case 4128: launch<4, 128>(ps, dir, keys, norm2_bits, s, cc); break;
    case 4256: launch<4, 256>(ps, dir, keys, norm2_bits, s, cc); break;
    case 8032: launch<8, 32>(ps, dir, keys, norm2_bits, s, cc); break;
    case 8064: launch<8, 64>(ps, dir, keys, norm2_bits, s, cc); break;
    case 8128: launch<8, 128>(ps, dir, keys, norm2_bits, s, cc); break;
    case 8256: launch<8, 256>(ps, dir, keys, norm2_bits, s, cc); break;
    default: throw std::logic_error("project_tc: unsupported shape");
  }
}

}  // namespace psg
