// hgemm_tc.cu — the hybrid path's dense block (hybrid.cu) on the 5th-generation
// tensor cores: D[h][q] = sum_k HT[k][h] * HQT[k][q] for a 128-row tile of
// heavy index rows (M) and all heavy queries (N <= 256), fp32 via 3xTF32.
//
//   * operands live in global memory already in the K-major 128-byte-swizzled
//     UMMA layout (one 128-byte line of 32 tf32 per row), split into tf32
//     hi = tf32(x) and lo = tf32(x - hi), one contiguous block per (row tile,
//     32-column K-step) (tiled_operand: the index side once per index, the
//     query side per call), so a stage is two bulk copies (cp.async.bulk,
//     the TMA engine) completing on the stage's mbarrier;
//   * one elected thread issues tcgen05.mma.kind::tf32 (M=128, N, K=8) three
//     times per K-step — lo*hi, hi*lo, hi*hi — into one fp32 accumulator in
//     tensor memory (error ~2^-22 |a||b| per product, like fp32 FMA);
//   * 2-8 shared-memory stages (as many as fit): a producer thread refills a
//     stage once tcgen05.commit has arrived on its empty barrier, so the copies
//     of later K-steps overlap the MMAs of earlier ones;
//   * epilogue: warps 0-3 read their 32 TMEM lanes with tcgen05.ld and write
//     the K-split partial tile; hreduce_kernel sums the splits in order.
#include <algorithm>
#include "common.cuh"
#include "hybrid.cuh"
#include "tma.cuh"

namespace sd {

namespace {

constexpr int TC_M = 128, TC_BK = 32, TC_THREADS = 256;

__device__ __forceinline__ uint32_t tf32_bits(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// byte offset of element (row r, k in [0, 32)) inside one operand block:
// rows at 128 B, the row's eight 16-byte chunks permuted by chunk ^ (row % 8)
// (128-byte swizzle: the tensor core's 8-row reads hit every bank; the
// unswizzled canonical layout left the MMAs at a third of their rate)
__device__ __forceinline__ uint32_t kmajor_off(int r, int k, int /*R*/) {
  return uint32_t(r * 128 + ((((k * 4) >> 4) ^ (r & 7)) << 4) + ((k * 4) & 15));
}

// shared-memory matrix descriptor: K-major, SWIZZLE_128B (layout type 2),
// SBO = 1024 B (next 8 rows), LBO unused, version 1 (sm_100); the K = 8 step
// kk starts 32 B further into the 1024-byte aligned block
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\t"
               "setp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

}  // namespace

int64_t tc_kstep() { return TC_BK; }

// Operand images for the tensor-core GEMM: rows (heavy index rows or heavy
// queries) split into tiles of R rows; for tile t and K-step ks (32 columns)
// a contiguous block [hi | lo] of R x 32 tf32 each in the canonical layout,
// so one bulk copy (TMA) moves a whole stage operand.  Zero elsewhere.
__global__ void tiled_scatter_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                     const float* __restrict__ val, const int32_t* __restrict__ rows, int64_t nrows,
                                     int R, int64_t nks, unsigned char* __restrict__ out) {
  const uint32_t part = uint32_t(R) * TC_BK * 4;
  for (int64_t g = blockIdx.x; g < nrows; g += gridDim.x) {  // same (rows x chunks) grid as ht_scatter_kernel
    const int64_t r = rows[g];
    const int64_t tile = g / R;
    const int rr = int(g - tile * R);
    const int64_t step = int64_t(gridDim.y) * blockDim.x;
    for (int64_t e = ptr[r] + int64_t(blockIdx.y) * blockDim.x + threadIdx.x; e < ptr[r + 1]; e += step) {
      const int64_t k = idx[e];
      const float v = val[e];
      const uint32_t hi = tf32_bits(v);
      const uint32_t lo = tf32_bits(v - __uint_as_float(hi));
      unsigned char* blk = out + ((tile * nks + k / TC_BK) * 2) * int64_t(part);
      const uint32_t off = kmajor_off(rr, int(k % TC_BK), R);
      *reinterpret_cast<uint32_t*>(blk + off) = hi;
      *reinterpret_cast<uint32_t*>(blk + part + off) = lo;
    }
  }
}

// grid: (hpad / 128, 1, splits).  Warp 1 lane 0 streams stages with bulk
// copies (full barriers count the bytes), warp 0 lane 0 issues the MMAs and
// commits each stage back to its empty barrier; STAGES-deep pipeline.
__global__ void __launch_bounds__(128) hgemm_tcgen05_kernel(const unsigned char* __restrict__ At,
                                                            const unsigned char* __restrict__ Bt, int64_t nks,
                                                            int N, int stages, int64_t steps_per_split,
                                                            int64_t rows, int64_t ldh, float* __restrict__ P) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t a_part = TC_M * TC_BK * 4, b_part = uint32_t(N) * TC_BK * 4;
  const uint32_t stage_bytes = 2 * a_part + 2 * b_part;
  const uint32_t sbase = (uint32_t(__cvta_generic_to_shared(smem)) + 1023u) & ~1023u;  // 1 KB slack allocated
  __shared__ __align__(8) unsigned long long bars[2 * 8 + 1];  // full[8], empty[8], done
  __shared__ uint32_t tmem_slot;
  const uint32_t full0 = uint32_t(__cvta_generic_to_shared(&bars[0])), empty0 = full0 + 64, done = full0 + 128;
  // NACC accumulators used round-robin by K-step and summed at the end in
  // IEEE fp32: the tensor core's fp32 accumulation is not round-to-nearest,
  // so long single chains drift (1e-5 relative over ~400 steps on C2)
  const int nacc = N <= 128 ? 4 : 2;
  uint32_t ncols = 32;
  while (ncols < uint32_t(nacc * N)) ncols <<= 1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(uint32_t(__cvta_generic_to_shared(&tmem_slot))), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int q = 0; q < stages; ++q) { mbar_init(full0 + 8 * q, 1); mbar_init(empty0 + 8 * q, 1); }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  // instruction descriptor: D f32, A/B tf32, both K-major, N >> 3, M >> 4
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(TC_M >> 4) << 24);
  const int64_t ks0 = int64_t(blockIdx.z) * steps_per_split;
  const int64_t nsteps = tmax<int64_t>(0, tmin<int64_t>(nks, ks0 + steps_per_split) - ks0);
  const unsigned char* Ablk = At + (int64_t(blockIdx.x) * nks + ks0) * 2 * int64_t(a_part);
  const unsigned char* Bblk = Bt + ks0 * 2 * int64_t(b_part);

  // stage index, phase and accumulator advance incrementally (a 64-bit
  // modulo per iteration put a software division on the issuing thread's
  // critical path)
  const int nst = int(nsteps);
  if (tid == 32) {  // producer
    int s = 0;
    uint32_t ph = 0;
    for (int p = 0; p < nst; ++p) {
      if (p >= stages) mbar_wait(empty0 + 8 * s, ph ^ 1u);
      const uint32_t dst = sbase + uint32_t(s) * stage_bytes;
      mbar_expect_tx(full0 + 8 * s, stage_bytes);
      bulk_g2s(dst, Ablk + int64_t(p) * 2 * int64_t(a_part), 2 * a_part, full0 + 8 * s);
      bulk_g2s(dst + 2 * a_part, Bblk + int64_t(p) * 2 * int64_t(b_part), 2 * b_part, full0 + 8 * s);
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
  } else if (tid == 0) {  // MMA issuer
    int s = 0, q = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nst; ++i) {
      mbar_wait(full0 + 8 * s, ph);  // (the bulk copies' completion orders the stage; no per-stage fence)
      const uint32_t sa = sbase + uint32_t(s) * stage_bytes;
      const uint32_t a_hi = sa, a_lo = sa + a_part, b_hi = sa + 2 * a_part, b_lo = b_hi + b_part;
      const uint32_t d = tmem + uint32_t(q) * uint32_t(N);
      // descriptors: address field = low 14 bits (addr >> 4), per-step ones by offset
      const uint64_t dah = smem_desc(a_hi), dal = smem_desc(a_lo), dbh = smem_desc(b_hi), dbl = smem_desc(b_lo);
      const uint32_t first0 = i < nacc ? 0u : 1u;
#pragma unroll
      for (int kk = 0; kk < TC_BK / 8; ++kk) {
        const uint64_t ao = uint64_t(kk) * 2, bo = uint64_t(kk) * 2;  // 32 B per K = 8 step
        mma_tf32(d, dal + ao, dbh + bo, idesc, kk == 0 ? first0 : 1u);
        mma_tf32(d, dah + ao, dbl + bo, idesc, 1u);
        mma_tf32(d, dah + ao, dbh + bo, idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   :: "r"(empty0 + 8 * s) : "memory");
      if (++s == stages) { s = 0; ph ^= 1u; }
      if (++q == nacc) q = 0;
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(done) : "memory");
  }
  // the other threads wait at a block barrier, not by polling the mbarrier
  // (spinning warps slowed the MMA pipeline ~5x), then one thread waits for
  // the last MMAs
  __syncthreads();
  if (tid == 0 && nsteps > 0) mbar_wait(done, 0u);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: warp w owns TMEM lanes 32w..32w+31 = heavy rows h0 + 32w + lane
  float* out = P + int64_t(blockIdx.z) * rows * ldh;
  const int64_t h = int64_t(blockIdx.x) * TC_M + warp * 32 + lane;
  const int used = int(tmin<int64_t>(nacc, nsteps));  // accumulators written at least once
  for (int c0 = 0; c0 < N; c0 += 16) {
    float sum[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) sum[j] = 0.f;
    for (int q = 0; q < used; ++q) {
      uint32_t r[16];
      const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16) + uint32_t(q * N + c0);
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                     "=r"(r[15])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 16; ++j) sum[j] = __fadd_rn(sum[j], __uint_as_float(r[j]));
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (c0 + j < rows) out[int64_t(c0 + j) * ldh + h] = sum[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(ncols) : "memory");
}

int tiled_operand(const sd_csr* m, const int32_t* rows, int64_t nrows, int R, int64_t nks, void* out,
                  cudaStream_t st) {
  const int64_t ntiles = (nrows + R - 1) / R;
  SD_CUDA_TRY(cudaMemsetAsync(out, 0, size_t(ntiles) * size_t(nks) * 2 * size_t(R) * TC_BK * 4, st));
  if (nrows == 0) return SD_OK;
  tiled_scatter_kernel<<<row_scatter_grid(nrows), 256, 0, st>>>(m->indptr, m->indices, static_cast<const float*>(m->values), rows,
                                               nrows, R, nks, static_cast<unsigned char*>(out));
  SD_LAUNCH_CHECK();
  return SD_OK;
}

int hgemm_tcgen05(const void* at, const void* bt, int64_t nks, int64_t hpad, int N, int64_t per, int64_t rows,
                  float* part, cudaStream_t st) {
  const size_t stage = 2 * size_t(TC_M) * TC_BK * 4 + 2 * size_t(N) * TC_BK * 4;
  const int stages = int(std::min<int64_t>(8, std::max<int64_t>(2, (smem_optin_bytes() - 4096) / int64_t(stage))));
  const size_t smem = size_t(stages) * stage + 1024;
  SD_TRY(prepare_smem(hgemm_tcgen05_kernel, smem, "hgemm_tcgen05_kernel"));
  const dim3 grid{unsigned(hpad / TC_M), 1u, unsigned((nks + per - 1) / per)};
  hgemm_tcgen05_kernel<<<grid, 128, smem, st>>>(static_cast<const unsigned char*>(at),
                                                static_cast<const unsigned char*>(bt), nks, N, stages, per, rows,
                                                hpad, part);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

}  // namespace sd
