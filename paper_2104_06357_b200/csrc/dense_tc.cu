// dense_tc.cu — dense-index mode: the whole distance matrix of a dot-family
// metric as one tensor-core GEMM with the metric fused into its epilogue.
//
// For dense-ish indexes (C4: 65,000 x 26,000 at ~7 % density, rows of
// 501-9,600 nonzeros) the intersection sweep does ~16 G posting updates for
// 2,048 queries (40 ms); the same sums as a dense GEMM, 2,048 x 65,000 x
// 26,000 multiply-adds, are ~7 TFLOP that the 5th-generation tensor cores run
// in a few milliseconds even at 3x the work for fp32-level accuracy:
//
//   * operand images (index: once per index; queries: per call) hold every
//     row as bf16 planes in the K-major 128-byte-swizzled UMMA layout, one
//     contiguous block per (128-row tile, 64-column K block) so a pipeline
//     stage is one bulk copy (TMA engine) per operand.  Rows whose values are
//     all bf16-exact (binary data: jaccard, dice, russelrao) keep one plane;
//     otherwise two, hi = bf16(x) and lo = bf16(x - hi) (|x - hi - lo| <=
//     2^-17 |x|);
//   * D[j][q] = sum_k A[j][k] B[q][k] with M = 128 index rows x N = 128
//     queries per CTA (256 for one-plane operands): tcgen05.mma.kind::f16 (bf16 in, fp32 accumulate in
//     tensor memory), hi*hi + hi*lo + lo*hi when both sides carry two planes
//     (the dropped lo*lo term is <= 2^-18 |a b|), issued by one thread; a
//     producer thread keeps 3-6 stages of bulk copies in flight on mbarriers;
//   * the tensor core's fp32 accumulation is not round-to-nearest, so K
//     blocks rotate over 4 accumulators (512 TMEM columns; 2 at N = 256,
//     where the sums are exact) that the epilogue sums in IEEE fp32;
//   * epilogue: warp w reads TMEM lanes 32w..32w+31 (index rows) with
//     tcgen05.ld, applies the metric's expansion with the rows' statistics
//     (expand_cell_t, the same function as every other path) and stores each
//     query's 32 cells as one 128-byte segment (streaming stores).
//
// Grid: (query tiles, index tiles), query tile fastest, so the CTAs that run
// together share their index tile through the L2.
#include <algorithm>
#include <cuda_bf16.h>
#include "common.cuh"
#include "hybrid.cuh"
#include "index.cuh"
#include "metric.cuh"
#include "prep.cuh"
#include "tma.cuh"

namespace sd {

namespace {

constexpr int DT_M = 128, DT_KB = 64;
constexpr uint32_t DT_PLANE = 128u * DT_KB * 2u;  // one bf16 plane of a 128-row x 64-column block (16 KB)
constexpr int DT_MAX_STAGES = 8;

// byte offset of (row r < 128, column k < 64) in a plane: K-major with the
// 128-byte swizzle — each row's 64 columns are one 128-byte line (rows at
// 128 B), its eight 16-byte chunks permuted by chunk ^ (row % 8), so the
// tensor core's reads of 8-row groups hit all banks (the unswizzled
// canonical layout put every 8-row group on the same banks: MMAs ran at a
// third of their rate)
__device__ __forceinline__ uint32_t kmajor16_off(int r, int k) {
  return uint32_t(r * 128 + ((((k * 2) >> 4) ^ (r & 7)) << 4) + ((k * 2) & 15));
}

// shared-memory matrix descriptor: K-major, SWIZZLE_128B (layout type 2),
// SBO = 1024 B between 8-row groups, LBO unused (1), version 1 (sm_100); the
// K = 16 step kk starts 32 B further into the (1024-byte aligned) tile
__device__ __forceinline__ uint64_t smem_desc16(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\t"
               "setp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// rows of a CSR into the image: [row tile of R][K block][plane][R x 128 B];
// the (rows x chunks) grid of the other scatter kernels
__global__ void dense_scatter_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                     const float* __restrict__ val, const int32_t* __restrict__ rows, int64_t nrows,
                                     int64_t nkb, int planes, int R, unsigned char* __restrict__ img) {
  const int64_t plane = int64_t(R) * DT_KB * 2;
  for (int64_t g = blockIdx.x; g < nrows; g += gridDim.x) {
    const int64_t tile = g / R;
    const int rr = int(g - tile * R);
    const int64_t src = rows ? int64_t(rows[g]) : g;  // image row g = CSR row src
    const int64_t step = int64_t(gridDim.y) * blockDim.x;
    for (int64_t e = ptr[src] + int64_t(blockIdx.y) * blockDim.x + threadIdx.x; e < ptr[src + 1]; e += step) {
      const int64_t k = idx[e];
      const float v = val[e];
      const __nv_bfloat16 hi = __float2bfloat16_rn(v);
      unsigned char* blk = img + (tile * nkb + (k >> 6)) * int64_t(planes) * plane;
      const uint32_t off = kmajor16_off(rr, int(k & 63));
      *reinterpret_cast<__nv_bfloat16*>(blk + off) = hi;
      if (planes == 2) *reinterpret_cast<__nv_bfloat16*>(blk + plane + off) = __float2bfloat16_rn(v - __bfloat162float(hi));
    }
  }
}

// flag bit 0: some value is not exactly representable in bf16; bit 1: some
// value is not a small integer (|v| <= 16)
__global__ void bf16_exact_kernel(const float* __restrict__ v, int64_t n, unsigned int* flag) {
  bool inexact = false, nonint = false;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const float x = v[e];
    inexact |= __bfloat162float(__float2bfloat16_rn(x)) != x;
    nonint |= !(fabsf(x) <= 16.f && rintf(x) == x);
  }
  // (block-wide votes: a warp-vote form of this was compiled into a wrong
  // exit predicate — it skipped the write exactly when both flags were set)
  const int any_inexact = __syncthreads_or(inexact), any_nonint = __syncthreads_or(nonint);
  if (threadIdx.x == 0 && (any_inexact || any_nonint)) atomicOr(flag, (any_inexact ? 1u : 0u) | (any_nonint ? 2u : 0u));
}

struct DenseArgs {
  const unsigned char* ai;  // index image (pa planes per block)
  const unsigned char* bq;  // query image (2 planes per block, pb of them loaded)
  int64_t nkb;
  int pa, pb;
  int64_t m, n, ldo;
  const float* sa0; const float* sa1; const float* sb0; const float* sb1;
  float k, p;
  float* out;
  uint32_t* flags;
  // RAW (the hybrid path's heavy block): K blocks [z*per, (z+1)*per) per
  // blockIdx.z, raw sums to part[z][q][h] (q < prow, h < ldp; zero padding included)
  int64_t per, prow, ldp;
  float* part;
};

// N queries per CTA (128, or 256 for one-plane operands): 512 / N accumulators
template <int M, int N, bool RAW>
__global__ void __launch_bounds__(128, 1) dense_tc_kernel(const DenseArgs a, int stages) {
  constexpr int NACC = 512 / N;
  constexpr uint32_t BPLANE = uint32_t(N) * DT_KB * 2u;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t a_bytes = uint32_t(a.pa) * DT_PLANE, b_bytes = uint32_t(a.pb) * BPLANE;
  const uint32_t stage_bytes = a_bytes + b_bytes;
  // the swizzle pattern repeats every 1024 B: stage bases 1024-aligned (1 KB of slack is allocated)
  const uint32_t sbase = (uint32_t(__cvta_generic_to_shared(smem)) + 1023u) & ~1023u;
  __shared__ __align__(8) unsigned long long bars[2 * DT_MAX_STAGES + 1];  // full, empty, done
  __shared__ uint32_t tmem_slot;
  __shared__ float qs0[N], qs1[N];  // the tile's query statistics, read by the epilogue
  for (int c = tid; c < N; c += blockDim.x) {
    const int64_t q = int64_t(blockIdx.x) * N + c;
    qs0[c] = q < a.m && a.sa0 ? a.sa0[q] : 0.f;
    qs1[c] = q < a.m && a.sa1 ? a.sa1[q] : 0.f;
  }
  const uint32_t full0 = uint32_t(__cvta_generic_to_shared(&bars[0])), empty0 = full0 + 8 * DT_MAX_STAGES,
                 done = full0 + 16 * DT_MAX_STAGES;
  constexpr uint32_t NCOLS = NACC * N;  // 512 TMEM columns
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(uint32_t(__cvta_generic_to_shared(&tmem_slot))), "r"(NCOLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int q = 0; q < stages; ++q) { mbar_init(full0 + 8 * q, 1); mbar_init(empty0 + 8 * q, 1); }
    mbar_init(done, 1);
    mbar_fence_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  // instruction descriptor: D f32, A/B bf16, both K-major, N >> 3, M >> 4
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(DT_M >> 4) << 24);
  const int64_t qt = blockIdx.x, jt = blockIdx.y;
  const int64_t kb0 = RAW ? int64_t(blockIdx.z) * a.per : 0;
  const unsigned char* Ablk = a.ai + (jt * a.nkb + kb0) * int64_t(a_bytes);
  const unsigned char* Bblk = a.bq + (qt * a.nkb + kb0) * int64_t(2 * BPLANE);
  // stage index and barrier phase advance incrementally: a 64-bit `p % stages`
  // per iteration (a software division on one thread's dependent chain)
  // cost ~0.4 us per stage, more than the MMAs themselves
  const int nkb = int(RAW ? tmin<int64_t>(a.per, a.nkb - kb0) : a.nkb);
  if (tid == 32) {  // producer
    int s = 0;
    uint32_t ph = 0;
    for (int p = 0; p < nkb; ++p) {
      if (p >= stages) mbar_wait(empty0 + 8 * s, ph ^ 1u);
      const uint32_t dst = sbase + uint32_t(s) * stage_bytes;
      mbar_expect_tx(full0 + 8 * s, stage_bytes);
      bulk_g2s(dst, Ablk + int64_t(p) * a_bytes, a_bytes, full0 + 8 * s);
      bulk_g2s(dst + a_bytes, Bblk + int64_t(p) * (2 * BPLANE), b_bytes, full0 + 8 * s);
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
  } else if (tid == 0) {  // MMA issuer
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nkb; ++i) {
      // (no tcgen05.fence per stage: the bulk copies' completion on the
      // mbarrier already orders the stage before the MMAs that read it; the
      // fence cost ~300 cycles per iteration of this single-thread loop)
      mbar_wait(full0 + 8 * s, ph);
      {
        const uint32_t sa = sbase + uint32_t(s) * stage_bytes, sb = sa + a_bytes;
        const uint32_t d = tmem + uint32_t(i & (NACC - 1)) * uint32_t(N);
        // descriptors: the address field is the low 14 bits (addr >> 4), so
        // the per-step ones are the stage's plus a small offset (the issuing
        // thread's instruction count per MMA bounded the one-plane case)
        const uint64_t da = smem_desc16(sa), db = smem_desc16(sb);
        const uint64_t dal = da + (DT_PLANE >> 4), dbl = db + (BPLANE >> 4);
        const uint32_t first0 = i < NACC ? 0u : 1u;
        if (a.pa == 1 && a.pb == 1) {
#pragma unroll
          for (int kk = 0; kk < DT_KB / 16; ++kk)
            mma_bf16(d, da + 2 * kk, db + 2 * kk, idesc, kk == 0 ? first0 : 1u);
        } else {
#pragma unroll
          for (int kk = 0; kk < DT_KB / 16; ++kk) {
            mma_bf16(d, da + 2 * kk, db + 2 * kk, idesc, kk == 0 ? first0 : 1u);   // hi * hi
            if (a.pb == 2) mma_bf16(d, da + 2 * kk, dbl + 2 * kk, idesc, 1u);     // hi * lo
            if (a.pa == 2) mma_bf16(d, dal + 2 * kk, db + 2 * kk, idesc, 1u);     // lo * hi
          }
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     :: "r"(empty0 + 8 * s) : "memory");
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(done) : "memory");
  }
  // the other threads wait at a block barrier, not by polling the mbarrier
  // (spinning warps slowed the MMA pipeline ~5x), then one thread waits for
  // the last MMAs
  __syncthreads();
  if (tid == 0 && nkb > 0) mbar_wait(done, 0u);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: warp w owns TMEM lanes 32w..32w+31 = index rows j
  const int64_t j = jt * DT_M + warp * 32 + lane;
  const bool jok = j < a.n;
  const float gb0 = jok && a.sb0 ? a.sb0[j] : 0.f, gb1 = jok && a.sb1 ? a.sb1[j] : 0.f;
  const int used = int(tmin<int64_t>(NACC, nkb));
  uint32_t flags = 0;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float sum[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) sum[c] = 0.f;
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
      for (int c = 0; c < 16; ++c) sum[c] = __fadd_rn(sum[c], __uint_as_float(r[c]));
    }
    if constexpr (RAW) {
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int64_t q = qt * N + c0 + c;
        if (q < a.prow && j < a.ldp) a.part[(int64_t(blockIdx.z) * a.prow + q) * a.ldp + j] = sum[c];
      }
      continue;
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int64_t q = qt * N + c0 + c;
      if (q < a.m && jok) {
        const float ra0 = qs0[c0 + c], ra1 = qs1[c0 + c];
        uint32_t f = 0;
        __stcs(a.out + q * a.ldo + j, expand_cell_t<M, float>(sum[c], ra0, ra1, gb0, gb1, a.k, a.p, f));
        flags |= f;
      }
    }
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (flags && lane == 0) atomicOr(a.flags, flags);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(NCOLS) : "memory");
}

template <int M, int N, bool RAW = false>
int launch_dense_n(const DenseArgs& a, cudaStream_t st, unsigned splits = 1) {
  // as many stages as fit: the stages stream from the L2, whose latency the
  // pipeline depth hides
  const size_t stage = size_t(a.pa) * DT_PLANE + size_t(a.pb) * size_t(N) * DT_KB * 2;
  const int stages = int(std::min<int64_t>(DT_MAX_STAGES, (smem_optin_bytes() - 6144) / int64_t(stage)));
  const size_t smem = size_t(stages) * stage + 1024;
  SD_TRY(prepare_smem(dense_tc_kernel<M, N, RAW>, smem, "dense_tc_kernel"));
  const dim3 grid{unsigned((a.m + N - 1) / N), unsigned((a.n + DT_M - 1) / DT_M), splits};
  dense_tc_kernel<M, N, RAW><<<grid, 128, smem, st>>>(a, stages);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

// small-integer operands on both sides (binary data: jaccard, dice,
// russelrao): 256 queries per CTA halve the index tile's L2 traffic per MMA,
// and every partial sum is an exact integer in fp32 (< 2^24 for K <= 65536),
// so two accumulators suffice.  Otherwise 128 queries and four accumulators
// (the tensor core's fp32 accumulation is not round-to-nearest; shorter
// chains per accumulator bound its drift).
int dense_tile_n(bool ints, int64_t n_cols) { return ints && n_cols <= 65536 ? 256 : 128; }

template <int M>
int launch_dense(const DenseArgs& a, int N, cudaStream_t st) {
  return N == 256 ? launch_dense_n<M, 256>(a, st) : launch_dense_n<M, 128>(a, st);
}

}  // namespace

int check_bf16_exact(const sd_csr* m, unsigned int* flag, cudaStream_t st) {
  if (m->nnz == 0) return SD_OK;
  const int blocks = int(tmin<int64_t>((m->nnz + 255) / 256, int64_t(num_sms()) * 8));
  bf16_exact_kernel<<<blocks, 256, 0, st>>>(static_cast<const float*>(m->values), m->nnz, flag);
  SD_LAUNCH_CHECK();
  return SD_OK;
}

namespace {

size_t image_bytes(int64_t rows, int64_t nkb, int planes, int R) {
  return size_t((rows + R - 1) / R) * size_t(nkb) * size_t(planes) * size_t(R) * DT_KB * 2;
}

int build_image(const sd_csr* m, const int32_t* rows, int64_t nrows, int64_t nkb, int planes, int R, void* img,
                cudaStream_t st) {
  SD_CUDA_TRY(cudaMemsetAsync(img, 0, image_bytes(nrows, nkb, planes, R), st));
  if (nrows == 0 || m->nnz == 0) return SD_OK;
  dense_scatter_kernel<<<row_scatter_grid(nrows), 256, 0, st>>>(m->indptr, m->indices,
                                                               static_cast<const float*>(m->values), rows, nrows,
                                                               nkb, planes, R, static_cast<unsigned char*>(img));
  SD_LAUNCH_CHECK();
  return SD_OK;
}

}  // namespace

// Dense-index mode applies to pairwise dot-family metrics in fp32 on an index
// of density >= 2 % whose image fits the memory budget (SD_TUNE_DENSE: 0 off,
// 1 automatic, 2 forced for any index — tests).
bool dense_eligible(const sd_csr* b, const sd_metric_desc* md, int dtype, int topk) {
  const int64_t kn = knob(SD_TUNE_DENSE);
  if (kn == 0 || topk != 0 || dtype != SD_F32 || metric_contrib(md->metric) != C_MUL) return false;
  if (b->n_rows == 0 || b->n_cols == 0) return false;
  if (kn == 2) return true;
  const double density = double(b->nnz) / (double(b->n_rows) * double(b->n_cols));
  const double img = double((b->n_rows + 127) / 128 * 128) * double((b->n_cols + 63) / 64 * 64) * 4.0;
  return density >= 0.02 && b->n_cols >= 256 && img <= double(knob(SD_TUNE_DENSE_MAX_MB)) * (1 << 20);
}

// index image (once per index): one plane when B is bf16-exact, else two
int ensure_dense(sd_index* ix, const sd_csr* b, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(ix->mu);
  if (ix->dimg) return SD_OK;
  Scratch flag;
  SD_TRY(flag.alloc(sizeof(unsigned int), st));
  SD_CUDA_TRY(cudaMemsetAsync(flag.ptr, 0, sizeof(unsigned int), st));
  SD_TRY(check_bf16_exact(b, flag.as<unsigned int>(), st));
  unsigned int inexact = 0;
  SD_CUDA_TRY(cudaMemcpyAsync(&inexact, flag.ptr, sizeof(inexact), cudaMemcpyDeviceToHost, st));
  SD_CUDA_TRY(cudaStreamSynchronize(st));
  const int planes = (inexact & 1u) ? 2 : 1;
  const int64_t nkb = (b->n_cols + DT_KB - 1) / DT_KB;
  const size_t bytes = image_bytes(b->n_rows, nkb, planes, DT_M);
  void* img = nullptr;
  if (cudaMalloc(&img, bytes) != cudaSuccess) {
    set_error("cudaMalloc failed for the dense index image");
    return SD_E_CUDA;
  }
  const int rc = build_image(b, nullptr, b->n_rows, nkb, planes, DT_M, img, st);
  if (rc != SD_OK) { cudaFree(img); return rc; }
  ix->dimg = img;
  ix->dplanes = planes;
  ix->dints = (inexact & 2u) == 0;
  ix->dnkb = nkb;
  ix->bytes += int64_t(bytes);
  return SD_OK;
}

int dense_run(const sd_csr* a, const sd_csr* b, const sd_index* ix, const sd_metric_desc* md, const Stats& sa,
              const Stats& sb, void* out, int64_t ldo, uint32_t* flags, cudaStream_t st) {
  if (a->n_rows == 0 || b->n_rows == 0) return SD_OK;
  if (a->n_cols != b->n_cols || ix->dnkb != (a->n_cols + DT_KB - 1) / DT_KB) {
    set_error("dense image does not match the operands");
    return SD_E_INVALID;
  }
  // query image: two planes in tiles of the CTA's query count (the lo plane
  // is loaded only if some query value is not bf16-exact)
  Scratch flag, img;
  SD_TRY(flag.alloc(sizeof(unsigned int), st));
  SD_CUDA_TRY(cudaMemsetAsync(flag.ptr, 0, sizeof(unsigned int), st));
  SD_TRY(check_bf16_exact(a, flag.as<unsigned int>(), st));
  unsigned int inexact = 0;
  SD_CUDA_TRY(cudaMemcpyAsync(&inexact, flag.ptr, sizeof(inexact), cudaMemcpyDeviceToHost, st));
  SD_CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t nkb = ix->dnkb;
  const int pb = (inexact & 1u) ? 2 : 1;
  const int R = dense_tile_n(ix->dints && (inexact & 2u) == 0, a->n_cols);
  SD_TRY(img.alloc(image_bytes(a->n_rows, nkb, 2, R), st));
  SD_TRY(build_image(a, nullptr, a->n_rows, nkb, 2, R, img.ptr, st));
  DenseArgs d;
  d.ai = static_cast<const unsigned char*>(ix->dimg);
  d.bq = static_cast<const unsigned char*>(img.ptr);
  d.nkb = nkb;
  d.pa = ix->dplanes;
  d.pb = pb;
  d.m = a->n_rows; d.n = b->n_rows; d.ldo = ldo;
  d.sa0 = static_cast<const float*>(sa.s[0]); d.sa1 = static_cast<const float*>(sa.s[1]);
  d.sb0 = static_cast<const float*>(sb.s[0]); d.sb1 = static_cast<const float*>(sb.s[1]);
  d.k = float(a->n_cols); d.p = float(md->p);
  d.out = static_cast<float*>(out);
  d.flags = flags;
  switch (md->metric) {
    case SD_M_CORRELATION: return launch_dense<SD_M_CORRELATION>(d, R, st);
    case SD_M_COSINE: return launch_dense<SD_M_COSINE>(d, R, st);
    case SD_M_DICE: return launch_dense<SD_M_DICE>(d, R, st);
    case SD_M_DOT: return launch_dense<SD_M_DOT>(d, R, st);
    case SD_M_EUCLIDEAN: return launch_dense<SD_M_EUCLIDEAN>(d, R, st);
    case SD_M_HELLINGER: return launch_dense<SD_M_HELLINGER>(d, R, st);
    case SD_M_JACCARD: return launch_dense<SD_M_JACCARD>(d, R, st);
    case SD_M_RUSSELRAO: return launch_dense<SD_M_RUSSELRAO>(d, R, st);
    default: set_error("metric has no dense-index mode"); return SD_E_UNSUPPORTED;
  }
}

// The hybrid path's heavy block on the same kernel (hybrid.cu): an image of
// rows `rows` of a CSR (nrows of them, tiles of R) ...
int64_t dense_kblocks(int64_t n_cols) { return (n_cols + DT_KB - 1) / DT_KB; }
size_t dense_image_bytes(int64_t nrows, int64_t nkb, int planes, int R) { return image_bytes(nrows, nkb, planes, R); }
int dense_image(const sd_csr* m, const int32_t* rows, int64_t nrows, int64_t nkb, int planes, int R, void* img,
                cudaStream_t st) {
  return build_image(m, rows, nrows, nkb, planes, R, img, st);
}

// ... and P[z][q][h] = sum over K blocks [z*per, (z+1)*per) of A_h . B_q for
// the index image A (na rows, pa planes, tiles of 128) and the query image B
// (nq rows, 2 planes stored, pb used, tiles of N = R), q < prow, h < ldp
int dense_gemm_raw(const void* aimg, int pa, int64_t na, const void* bimg, int pb, int R, int64_t nq, int64_t nkb,
                   int64_t per, float* part, int64_t prow, int64_t ldp, cudaStream_t st) {
  DenseArgs d{};
  d.ai = static_cast<const unsigned char*>(aimg);
  d.bq = static_cast<const unsigned char*>(bimg);
  d.nkb = nkb;
  d.pa = pa;
  d.pb = pb;
  d.m = nq; d.n = na;
  d.per = per; d.prow = prow; d.ldp = ldp; d.part = part;
  const unsigned splits = unsigned((nkb + per - 1) / per);
  return R == 256 ? launch_dense_n<SD_M_DOT, 256, true>(d, st, splits) : launch_dense_n<SD_M_DOT, 128, true>(d, st, splits);
}

}  // namespace sd
