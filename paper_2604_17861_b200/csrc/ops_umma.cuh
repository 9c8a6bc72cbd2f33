// Small-GEMM task body on the 5th-generation tensor cores (tcgen05), the one
// task type that uses them (north star): bf16/f16 matmul_small tasks
// (reference ops.hpp:363-433, dims <= 256 on the queued path).
//
// Per (128 x 128) output tile of one task, inside the executor group that
// runs it:
//   1. the group stages A (128 x 64 chunk of K) and B^T (128 x 64) from the
//      task's strided views into shared memory in the UMMA canonical K-major,
//      no-swizzle layout (8-row x 16-byte core matrices), zero-padding ragged
//      edges -- views are arbitrary strided tensors, so this is a gather,
//      not a TMA box;
//   2. one elected thread issues 4 x tcgen05.mma.cta_group::1.kind::f16
//      (M=128, N=128, K=16 each) accumulating in the group's 128 TMEM columns,
//      and tcgen05.commit arrives on the group's mbarrier;
//   3. after the last K chunk, each warp reads its 32-lane TMEM quadrant with
//      tcgen05.ld.32x32b and stores rounded bf16/f16 outputs.
//
// Numerics: bf16/f16 products are exact in fp32, accumulation is fp32 in the
// tensor core, one rounding to the output dtype at the end.  The reference
// accumulates in fp64 (ascending k); tests bound the difference by the fp32
// accumulation error (tests/parity.py rule "gemm32").
#pragma once

#include "dev_common.cuh"

namespace gdev {

constexpr int kUmmaM = 128, kUmmaN = 128, kUmmaKChunk = 64;
constexpr uint32_t kUmmaTileBytes = kUmmaM * kUmmaKChunk * 2;  // 16 KB per operand chunk

// UMMA shared-memory matrix descriptor, K-major, SWIZZLE_NONE (cute
// UMMA::SmemDescriptor): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version 1 [46,48), layout type 0 [61,64).
__device__ __forceinline__ uint64_t umma_smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}

// Instruction descriptor (cute UMMA::InstrDescriptor): F32 accumulate,
// A/B format (0 = F16, 1 = BF16), both K-major, N>>3 at [17,23), M>>4 at [24,29).
__device__ __forceinline__ uint32_t umma_instr_desc(int fmt, int m, int n) {
  return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void umma_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(mbar)),
               "r"(count)
               : "memory");
}

// TMEM allocation by one full warp; writes the base address to *dst (smem).
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 16 consecutive fp32 accumulator columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Canonical K-major no-swizzle placement of element (row, kk) of a
// rows x 64 chunk: 16-byte chunk index = (kk/8) * rows + row; element
// kk%8 inside it.  LBO (K direction) = rows*16 B, SBO (8-row groups) = 128 B.
__device__ __forceinline__ uint32_t umma_elem_off(int row, int kk, int rows) {
  return (uint32_t)(((kk >> 3) * rows + row) * 16 + (kk & 7) * 2);
}

// Gather a `rows` x 64 operand chunk into the canonical layout: element
// (r, kk) = src[(r0 + r) * s_r + (k0 + kk) * s_k], zero outside r < r_lim,
// k0 + kk < k_lim.  K-contiguous sources move one 16-byte core-matrix row per
// load; row-contiguous sources move eight rows of one k per load; anything
// else goes element by element -- in every case eight independent loads per
// thread are in flight before the first store.
__device__ __forceinline__ void umma_stage(char* dst, int rows, const uint16_t* src, int64_t s_r, int64_t s_k,
                                           int r0, int r_lim, int k0, int k_lim, const Ctx* c) {
  const int nt = c->nthreads;
  const bool base16 = ((uintptr_t)src & 15) == 0;
  if (s_k == 1 && base16 && (s_r & 7) == 0) {
    const int units = rows * (kUmmaKChunk / 8);
    for (int u0 = c->tid; u0 < units; u0 += nt * 8) {
      uint4 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int u = u0 + q * nt;
        v[q] = make_uint4(0, 0, 0, 0);
        if (u < units) {
          const int r = u >> 3, kc = u & 7;
          const int gr = r0 + r, gk = k0 + 8 * kc;
          if (gr < r_lim && gk + 8 <= k_lim) {
            v[q] = __ldcg(reinterpret_cast<const uint4*>(src + gr * s_r + gk));
          } else if (gr < r_lim && gk < k_lim) {
            uint16_t h[8];
            for (int i = 0; i < 8; ++i) h[i] = gk + i < k_lim ? __ldcg(src + gr * s_r + gk + i) : (uint16_t)0;
            v[q] = make_uint4(h[0] | ((uint32_t)h[1] << 16), h[2] | ((uint32_t)h[3] << 16), h[4] | ((uint32_t)h[5] << 16),
                              h[6] | ((uint32_t)h[7] << 16));
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int u = u0 + q * nt;
        if (u < units) {
          const int r = u >> 3, kc = u & 7;
          *reinterpret_cast<uint4*>(dst + (kc * rows + r) * 16) = v[q];
        }
      }
    }
    return;
  }
  if (s_r == 1 && base16 && (s_k & 7) == 0) {
    const int rg = rows / 8, units = rg * kUmmaKChunk;
    for (int u0 = c->tid; u0 < units; u0 += nt * 8) {
      uint4 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int u = u0 + q * nt;
        v[q] = make_uint4(0, 0, 0, 0);
        if (u < units) {
          const int g = u % rg, kk = u / rg;
          const int gr = r0 + 8 * g, gk = k0 + kk;
          if (gk < k_lim && gr + 8 <= r_lim) {
            v[q] = __ldcg(reinterpret_cast<const uint4*>(src + gr + gk * s_k));
          } else if (gk < k_lim && gr < r_lim) {
            uint16_t h[8];
            for (int i = 0; i < 8; ++i) h[i] = gr + i < r_lim ? __ldcg(src + gr + i + gk * s_k) : (uint16_t)0;
            v[q] = make_uint4(h[0] | ((uint32_t)h[1] << 16), h[2] | ((uint32_t)h[3] << 16), h[4] | ((uint32_t)h[5] << 16),
                              h[6] | ((uint32_t)h[7] << 16));
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int u = u0 + q * nt;
        if (u < units) {
          const int g = u % rg, kk = u / rg;
          const uint32_t w[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
          for (int i = 0; i < 8; ++i)
            *(uint16_t*)(dst + umma_elem_off(8 * g + i, kk, rows)) = (uint16_t)(w[i >> 1] >> (16 * (i & 1)));
        }
      }
    }
    return;
  }
  const int units = rows * kUmmaKChunk;
  for (int u0 = c->tid; u0 < units; u0 += nt * 8) {
    uint16_t v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int u = u0 + q * nt;
      const int r = u / kUmmaKChunk, kk = u % kUmmaKChunk;
      const int gr = r0 + r, gk = k0 + kk;
      v[q] = (u < units && gr < r_lim && gk < k_lim) ? __ldcg(src + gr * s_r + gk * s_k) : (uint16_t)0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int u = u0 + q * nt;
      if (u < units) *(uint16_t*)(dst + umma_elem_off(u / kUmmaKChunk, u % kUmmaKChunk, rows)) = v[q];
    }
  }
}

// out (m x n) = a (m x k) . b (k x n) for 16-bit float views, fp32 accumulate.
// Requires Ctx::tmem (128 columns) and Ctx::mbar; 32 KB of scratch.
__device__ int matmul_umma(const gpuos_view& a, const gpuos_view& b, const gpuos_view& out, int m, int k, int n,
                           const Ctx* c) {
  const int dt = out.dtype;
  const int fmt = dt == GPUOS_BF16 ? 1 : 0;
  const uint16_t* ap = (const uint16_t*)a.addr;
  const uint16_t* bp = (const uint16_t*)b.addr;
  char* sA = c->smem;
  char* sB = c->smem + kUmmaTileBytes;
  const uint32_t saA = (uint32_t)__cvta_generic_to_shared(sA);
  const uint32_t saB = (uint32_t)__cvta_generic_to_shared(sB);
  const int64_t sa0 = a.strides[0], sa1 = a.strides[1], sb0 = b.strides[0], sb1 = b.strides[1];
  const int64_t so0 = out.strides[0], so1 = out.strides[1];
  const int nt = c->nthreads;
  const int warp = c->tid >> 5, lane = c->tid & 31;
  // this thread's TMEM lane quadrant is fixed by its hardware warp id
  const int hw_warp = (int)(threadIdx.x >> 5);
  const int quad = hw_warp & 3;
  const int nwarps = nt >> 5;
  uint32_t phase = *c->mma_phase;
  const int ntm = (m + kUmmaM - 1) / kUmmaM, ntn = (n + kUmmaN - 1) / kUmmaN;
  int64_t tlo, thi;
  part_range((int64_t)ntm * ntn, c->part, c->nparts, 1, &tlo, &thi);
  for (int64_t tile = tlo; tile < thi; ++tile) {
    const int i0 = (int)(tile / ntn) * kUmmaM, j0 = (int)(tile % ntn) * kUmmaN;
    const int nn = (n - j0) < kUmmaN ? (n - j0) : kUmmaN;
    const int nmma = (nn + 15) & ~15;  // MMA N: multiple of 16
    const uint32_t idesc = umma_instr_desc(fmt, kUmmaM, nmma);
    for (int k0 = 0; k0 < k; k0 += kUmmaKChunk) {
      // stage A chunk (rows i0.., cols k0..) and B^T chunk (row j of the
      // N x K operand = column j0+j of b), zero beyond m / n / k
      umma_stage(sA, kUmmaM, ap, sa0, sa1, i0, m, k0, k, c);
      umma_stage(sB, kUmmaN, bp, sb1, sb0, j0, n, k0, k, c);
      // generic-proxy smem writes -> visible to the tensor core's async proxy
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      group_sync(c);
      tc_fence_after();
      if (c->tid == 0) {
#pragma unroll
        for (int s = 0; s < kUmmaKChunk / 16; ++s) {
          // K step s covers 16-byte chunks kc = 2s, 2s+1
          const uint64_t adesc = umma_smem_desc(saA + (uint32_t)(2 * s * kUmmaM * 16), kUmmaM * 16, 128);
          const uint64_t bdesc = umma_smem_desc(saB + (uint32_t)(2 * s * kUmmaN * 16), kUmmaN * 16, 128);
          umma_mma(c->tmem, adesc, bdesc, idesc, (k0 > 0 || s > 0) ? 1u : 0u);
        }
        umma_commit(c->mbar);
      }
      // wait for the MMAs (they read sA/sB) before the next chunk overwrites them
      mbar_wait(c->mbar, phase);
      phase ^= 1u;
      tc_fence_after();
    }
    // epilogue: this thread's row = 32*quad + lane; warps sharing a quadrant
    // split the columns
    const int row = 32 * quad + lane;
    const int sharers = nwarps >= 4 ? nwarps / 4 : 1;
    const int part_id = warp / 4;
    const int gi = i0 + row;
    for (int col0 = part_id * 16; col0 < nmma; col0 += 16 * sharers) {
      float v[16];
      tmem_ld16(c->tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)col0, v);
      if (gi < m) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int gj = j0 + col0 + q;
          if (col0 + q < nn) {
            uint16_t bits;
            if (dt == GPUOS_BF16) {
              const __nv_bfloat16 h = __float2bfloat16_rn(v[q]);
              bits = *reinterpret_cast<const uint16_t*>(&h);
            } else {
              const __half h = __float2half_rn(v[q]);
              bits = *reinterpret_cast<const uint16_t*>(&h);
            }
            *((uint16_t*)out.addr + gi * so0 + gj * so1) = bits;
          }
        }
      }
    }
    // every lane's TMEM reads done before the next tile's MMAs overwrite it
    tc_fence_before();
    group_sync(c);
    tc_fence_after();
  }
  if (c->tid == 0) *c->mma_phase = phase;
  return GPUOS_OK;
}

}  // namespace gdev
