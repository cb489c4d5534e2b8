// pair.cuh -- one thread-block cluster per image pair (images that fit in a
// cluster's shared memory; the band kernel handles larger ones).
//
// Replaces the body of Sampler._render_batch (reference pipeline.py:278-329)
// for such images: sample_particles / perturb_frame2 / advect / apply_hiding
// (particles.py:61-147), patch_side with the pair's maximum diameter
// (raster.py:30-38, pipeline.py:291-294), splat (raster.py:108-126 ->
// _native.pyx:14-66), finalize (raster.py:154-161), quantize_u16
// (export.py:19-20).
//
// Design (B200-first):
//   * A cluster of C CTAs owns one pair at a time; CTA k owns image rows
//     [k RB, (k + 1) RB) of both frames as an int32 fixed-point accumulator
//     in its shared memory. The C CTAs together hold the whole pair on chip.
//   * Phase A: the cluster's threads generate the M particles (index-strided,
//     each exactly once: Philox4x32-10 keyed by (particle, pair, batch,
//     stream), positions iid uniform over the image -- the reference's law,
//     particles.py:72-76 -- diameters iid uniform, advection). Every
//     particle-frame whose window reaches a CTA's rows becomes a 16-byte
//     (32 with correlation / sigma jitter) record stored straight into that
//     CTA's shared-memory inbox over DSMEM (st.shared::cluster): private
//     per-source regions, local slot counters, no remote atomics. Regions
//     that fill up spill to an L2-resident global buffer (exact, just slower).
//   * cluster barrier (release/acquire): the inbox, its counts and the other
//     CTAs' maximum diameters are visible. The pair's patch side follows from
//     the maximum diameter -- known now because every particle was generated.
//   * Phase B: each CTA splats its inbox into its rows (integer shared-memory
//     atomics: associative, so every pixel is bit-identical for any schedule,
//     cluster size or GPU count), then arrives on the cluster barrier (its
//     inbox may be refilled) and
//   * Phase C: finalizes and stores its rows of both frames (offset, Philox
//     noise, clamp, optional uint16; 128-bit streaming stores), zeroing the
//     accumulator, while the barrier completes.
// No prologue, no histogram, no regeneration: every particle is generated
// once and never leaves the chip; HBM traffic = the images.
#pragma once
#include "band.cuh"

namespace pgb {

constexpr int kPairThreads = 384;            // 12 warps; two CTAs per SM (<= 85 registers)
constexpr int kPairMaxCluster = 8;           // portable cluster size

__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// Shared-memory address of the same variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t cl_map(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((uint32_t)__cvta_generic_to_shared(local)),
               "r"(rank));
  return r;
}
__device__ __forceinline__ void cl_st4(uint32_t addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void cl_st1(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// One generated particle of the pair law: frame-1 position X / 2^17 (Q17,
// uniform over [0, W) x [0, H), particles.py:72-76) kept as Q20; frame-2
// position = frame-1 + rint(flow * 2^20) (64-bit: far displacements stay exact).
struct PairPart {
  int xq1, yq1;
  long long xq2, yq2;
  float d, sig;
  Look lk;
};

__device__ __forceinline__ void pair_particle(const GenCfg& g, const RngKey& key, int gi,
                                              const float2* __restrict__ flow, PairPart& o) {
  const uint4 a = philox_rk(make_uint4((uint32_t)gi, key.pair, key.batch, kTagParticleA), g.rk);
  const uint32_t X = cell_coord(0u, a.x, g.W, 0);
  const uint32_t Y = cell_coord(0u, a.y, g.H, 0);
  // advect (particles.py:129-136): bilinear, edge-clamped (flowfield.py:207-232);
  // fcx <= W - 2 and fcy <= H - 2, so the nodes are fp[0], fp[1], fp[W], fp[W + 1]
  int fcx, fcy;
  float tx, ty;
  fixed_cell(X, g.W, fcx, tx);
  fixed_cell(Y, g.H, fcy, ty);
  const float2* fp = flow + (fcy * g.W + fcx);
  const float2* fq = fp + g.W;
  const float2 q00 = __ldg(fp), q01 = __ldg(fp + 1);
  const float2 q10 = __ldg(fq), q11 = __ldg(fq + 1);
  o.d = lerpf_exact(g.d_lo, g.d_span, unit23(a.z));
  const float i0 = lerpf_exact(g.i0_lo, g.i0_span, unit23(a.w));
  o.sig = __fmul_rn(o.d, g.inv_ratio);
  seed_look(g, key, gi, o.sig, i0, o.lk);
  const float u = bilerp(q00.x, q01.x, q10.x, q11.x, tx, ty);
  const float v = bilerp(q00.y, q01.y, q10.y, q11.y, tx, ty);
  o.xq1 = (int)(X << 3);
  o.yq1 = (int)(Y << 3);
  o.xq2 = (long long)o.xq1 + __float2ll_rn(u * 1048576.0f);
  o.yq2 = (long long)o.yq1 + __float2ll_rn(v * 1048576.0f);
}

// Q20 -> anchor floor(v + 1/2) and the exact float32 fraction in [-1/2, 1/2).
__device__ __forceinline__ void q20_anchor(int q, int& a, float& f) {
  a = (q + (1 << 19)) >> 20;
  f = (float)(q - (a << 20)) * 0x1p-20f;
}

// Record words: SIMPLE (rho = 0, sx = sy: one uint4) {xq, yq, sigma, amp};
// full (two uint4) {xq, yq, sx, sy} {rho, amp, 0, 0}.
template <bool SIMPLE>
struct RecW {
  static constexpr int kWords = SIMPLE ? 1 : 2;
};

// Byte offsets of the shared-memory regions (identical in every CTA). The
// inbox, its counts and the maximum diameters are double-buffered: pair k+1
// is generated into buffer (k+1)&1 while buffer k&1 is being splatted.
struct PairSmem {
  int acc_ints;     // (frames RB + pad_rows) AS + 8
  int inbox_off;    // bytes: [2 buffers][2 frames][C sources][cap] records
  int cnt_in_off;   // [2][2][C] ints (written by the sources)
  int dmax_in_off;  // [2][C] floats (written by the sources)
  int cnt_out_off;  // [2][C] ints (this CTA's slot counters)
  int total;
  int buf_words;    // uint4 words per inbox buffer
};

// frames 2: both frame accumulators live at once; 1: one accumulator, frames in turn.
__host__ __device__ __forceinline__ PairSmem pair_smem(int rows, int pad_rows, int AS, int C, int cap, int words,
                                                       int frames = 1) {
  PairSmem s;
  s.acc_ints = (frames * rows + pad_rows) * AS + 8;
  s.inbox_off = ((s.acc_ints * 4) + 15) & ~15;
  s.buf_words = 2 * C * cap * words;
  s.cnt_in_off = s.inbox_off + 2 * s.buf_words * 16;
  s.dmax_in_off = s.cnt_in_off + 2 * 2 * C * 4;
  s.cnt_out_off = s.dmax_in_off + 2 * C * 4;
  s.total = ((s.cnt_out_off + 2 * C * 4) + 15) & ~15;
  return s;
}

// Per-pair splat parameters (thread 0 computes, shared with the block).
struct PairItem {
  int h, shift[2], var;
  int K[2];                 // records per frame (inbox + overflow)
  int kin[2];               // records per frame in the shared-memory inbox
  int pre[2][kPairMaxCluster + 1];   // inbox prefix over sources
  float inv_scale[2];
  float dmax;
  int side;
};

// One record into CTA `dst`'s inbox region of this source (local slot
// counter, then a DSMEM store); a full region spills to the destination's
// global overflow list of this frame (L2; exact, slower).
template <bool SIMPLE>
__device__ __forceinline__ void pair_emit(const BandParams& P, uint4* my_box, int* cnt_out, int f, int dst,
                                          const uint4& w0, const uint4& w1, int* ovf_cnt, uint4* ovf) {
  constexpr int RW = RecW<SIMPLE>::kWords;
  const int slot = atomicAdd(cnt_out + f * P.cl_size + dst, 1);
  if (slot < P.cl_cap) {
    const uint32_t ra = cl_map(my_box + (size_t)(f * P.cl_size * P.cl_cap + slot) * RW, (uint32_t)dst);
    cl_st4(ra, w0);
    if (!SIMPLE) cl_st4(ra + 16, w1);
  } else {
    const int o = atomicAdd(ovf_cnt + dst * 2 + f, 1);
    uint4* dp = ovf + ((size_t)(dst * 2 + f) * P.n + o) * RW;
    __stcg(dp, w0);
    if (!SIMPLE) __stcg(dp + 1, w1);
  }
}

// Route one particle-frame (Q20 position) to the CTAs owning the rows its
// tight window (anchor offsets within +-cl_hcfg) can touch. Windows that miss
// the image rows produce no record; the columns are clipped at splat time.
template <bool SIMPLE>
__device__ __forceinline__ void pair_route(const BandParams& P, uint4* my_box, int* cnt_out, int f,
                                           long long xq, long long yq, float sx, float sy, float rho, float amp,
                                           int* ovf_cnt, uint4* ovf) {
  const int hc = P.cl_hcfg;
  const long long ayl = (yq + (1 << 19)) >> 20, axl = (xq + (1 << 19)) >> 20;
  if (ayl < -hc - 1 || ayl > P.H + hc || axl < -hc - 1 || axl > P.W + hc) return;
  const int ay = (int)ayl;
  const float fy = (float)((int)yq - (ay << 20)) * 0x1p-20f;
  float R = __fmul_rn(fmaxf(sx, sy), kTightR);
  if (P.psf != kPsfPoint) R = __fadd_rn(R, 0.5f);
  const int lo = max(ay + max(-hc, (int)ceilf(__fsub_rn(fy, R))), 0);
  const int hi = min(ay + min(hc, (int)floorf(__fadd_rn(fy, R))), P.H - 1);
  if (lo > hi) return;
  const uint4 w0 = SIMPLE ? make_uint4((uint32_t)(int)xq, (uint32_t)(int)yq, __float_as_uint(sx), __float_as_uint(amp))
                          : make_uint4((uint32_t)(int)xq, (uint32_t)(int)yq, __float_as_uint(sx), __float_as_uint(sy));
  const uint4 w1 = make_uint4(__float_as_uint(rho), __float_as_uint(amp), 0u, 0u);
  const int d0 = (int)(((uint32_t)lo * P.cl_rdiv) >> 20), d1 = (int)(((uint32_t)hi * P.cl_rdiv) >> 20);
  pair_emit<SIMPLE>(P, my_box, cnt_out, f, d0, w0, w1, ovf_cnt, ovf);
  for (int d = d0 + 1; d <= d1; ++d) pair_emit<SIMPLE>(P, my_box, cnt_out, f, d, w0, w1, ovf_cnt, ovf);
}

// Phase B: splat this CTA's records of frame f (variant fixed per pair).
// Thread t takes records t, t + NT, ...: its source region index only moves
// forward (a running search over the inbox prefix).
template <int PSF, int SEP, int WM, bool SIMPLE>
__device__ __forceinline__ void pair_splat_frame(const BandParams& P, const uint4* inbox, int* acc,
                                                 const PairItem& it, int f, int r0, int r1, const uint4* ovf_f) {
  constexpr int RW = RecW<SIMPLE>::kWords;
  const int C = P.cl_size;
  const int kin = it.kin[f], K = it.K[f];
  const int shift = it.shift[f];
  const float scale = (float)(1 << shift);
  const int* pre = it.pre[f];
  int s = 0;
  int next = C > 1 ? pre[1] : 0x7fffffff;
  for (int q = threadIdx.x; q < K; q += kPairThreads) {
    const uint4* rp;
    if (q < kin) {
      while (q >= next) {
        ++s;
        next = s + 1 < C ? pre[s + 1] : 0x7fffffff;
      }
      rp = inbox + ((size_t)(f * C + s) * P.cl_cap + (q - pre[s])) * RW;
    } else {
      rp = ovf_f + (size_t)(q - kin) * RW;
    }
    uint4 w0, w1 = make_uint4(0u, 0u, 0u, 0u);
    if (q < kin) {
      w0 = rp[0];
      if (!SIMPLE) w1 = rp[1];
    } else {
      w0 = __ldcg(rp);
      if (!SIMPLE) w1 = __ldcg(rp + 1);
    }
    int ax, ay;
    float fx, fy;
    q20_anchor((int)w0.x, ax, fx);
    q20_anchor((int)w0.y, ay, fy);
    const float sx = __uint_as_float(w0.z);
    const float sy = SIMPLE ? sx : __uint_as_float(w0.w);
    const float rho = SIMPLE ? 0.f : __uint_as_float(w1.x);
    const float amp = SIMPLE ? __uint_as_float(w0.w) : __uint_as_float(w1.y);
    splat_v<PSF, SEP, WM>(acc, P.AS, ax, ay, fx, fy, amp, sx, sy, rho, it.h, r0, r1, 0, P.W, shift, scale);
  }
}

// Kernel variants: PSF, record format, and the particle loop's window bound
// WM (1..kPairMaxWM: unpredicated separable windows; 0: dynamic loops),
// chosen per launch from the configuration (the largest sigma any pair can
// have), so every kernel carries only the registers its variant needs.
constexpr int kPairMaxWM = 8;

// Rows [r0, r0 + nr) of frame f from the accumulator to the output
// (finalize, optional uint16), zeroing it; kPairThreads threads.
__device__ __forceinline__ void pair_store(const BandParams& P, int* acc, int pl, int f, int r0, int nr,
                                           float inv_scale) {
  if (nr <= 0) return;
  if ((P.W & 3) == 0 && P.AS == P.W) {
    const bool noise = P.noise_std > 0.f;
    const int t = threadIdx.x;
    switch (P.out_mode) {
      case kOutRaw: band_store_lin<kOutRaw, false>(P, acc, pl, f, r0, nr, inv_scale, t, kPairThreads); return;
      case kOutF32:
        if (noise) band_store_lin<kOutF32, true>(P, acc, pl, f, r0, nr, inv_scale, t, kPairThreads);
        else band_store_lin<kOutF32, false>(P, acc, pl, f, r0, nr, inv_scale, t, kPairThreads);
        return;
      default:
        if (noise) band_store_lin<kOutU16, true>(P, acc, pl, f, r0, nr, inv_scale, t, kPairThreads);
        else band_store_lin<kOutU16, false>(P, acc, pl, f, r0, nr, inv_scale, t, kPairThreads);
        return;
    }
  }
  // widths that are not a multiple of 4: one pixel per thread
  const uint32_t gpair = (uint32_t)(P.pair_base + pl);
  const size_t pair_off = (size_t)pl * (size_t)P.out_pair_elems;
  const int total = nr * P.W;
  for (int e = threadIdx.x; e < total; e += kPairThreads) {
    const int row = e / P.W, col = e - (e / P.W) * P.W;
    int* ap = acc + row * P.AS + col;
    float v = (float)*ap * inv_scale;
    *ap = 0;
    const size_t p = (size_t)(r0 + row) * P.W + (size_t)col;
    if (P.out_mode == kOutRaw) {
      static_cast<float*>(P.out[f])[pair_off + p] = v;
    } else {
      float nzv = 0.f;
      if (P.noise_std > 0.f) {
        const float4 nz = noise4_rk(P.g.rk, gpair, P.batch_lo, (uint32_t)f + 1, (uint32_t)(p >> 2));
        const int jn = (int)(p & 3);
        nzv = jn == 0 ? nz.x : (jn == 1 ? nz.y : (jn == 2 ? nz.z : nz.w));
      }
      v = finalize_px(v, P.bg_offset, P.noise_std, nzv);
      if (P.out_mode == kOutF32) static_cast<float*>(P.out[f])[pair_off + p] = v;
      else static_cast<uint16_t*>(P.out[f])[pair_off + p] = quant_u16(v);
    }
  }
}

template <bool SIMPLE>
struct PairCtx {
  int C, k;
  unsigned char* smem;
  PairSmem L;
  int* cnt_out;
  int* ovf_cnt;   // this cluster's [2 buffers][C][2]
  uint4* ovf;     // this cluster's [2 buffers][C][2][n] records
};

// Phase A of pair `pl` into inbox buffer b: generate this CTA's share of the
// particles and route their records; publish counts and the maximum diameter.
template <bool SIMPLE>
__device__ __forceinline__ void pair_phase_a(const BandParams& P, const PairCtx<SIMPLE>& X, int pl, int b,
                                             int* s_M, double* s_ppp, unsigned* s_dmax) {
  constexpr int RW = RecW<SIMPLE>::kWords;
  const GenCfg& g = P.g;
  const int tid = threadIdx.x, lane = tid & 31;
  const int C = X.C, k = X.k;
  const RngKey key = band_key(P, pl);
  if (tid == 0) {
    // seeding density and active count (particles.py:73-83)
    const uint4 w0 = philox_rk(make_uint4(0u, key.pair, key.batch, kTagPair), g.rk);
    const double ppp = lerp_exact(g.ppp_lo, g.ppp_hi, u53_to_unit(w0.x, w0.y));
    double mm = rint(dmul(dmul(ppp, (double)g.H), (double)g.W));
    mm = fmin(fmax(mm, 0.0), (double)P.n);
    s_M[b] = (int)mm;
    s_ppp[b] = ppp;
    *s_dmax = 0u;
  }
  __syncthreads();
  const int M = s_M[b];
  const float2* flow = P.flows + (size_t)((P.pair_base + pl) / P.pairs_per_field) * P.field_elems;
  uint4* my_box = reinterpret_cast<uint4*>(X.smem + X.L.inbox_off) + (size_t)b * X.L.buf_words +
                  (size_t)k * P.cl_cap * RW;   // [b][f = 0][k] region
  int* ovf_cnt = X.ovf_cnt + b * C * 2;
  uint4* ovf = X.ovf + (size_t)b * C * 2 * P.n * RW;
  unsigned dloc = 0u;
  for (int gi = k * kPairThreads + tid; gi < M; gi += C * kPairThreads) {
    PairPart pp;
    pair_particle(g, key, gi, flow, pp);
    dloc = max(dloc, __float_as_uint(pp.d));   // d >= 0: float order == bit order
    const Look& lk = pp.lk;
    if (lk.vis1 && lk.amp1 > 0.f)
      pair_route<SIMPLE>(P, my_box, X.cnt_out, 0, pp.xq1, pp.yq1, pp.sig, pp.sig, lk.rho1, lk.amp1, ovf_cnt, ovf);
    if (lk.vis2 && lk.amp2 > 0.f)
      pair_route<SIMPLE>(P, my_box, X.cnt_out, 1, pp.xq2, pp.yq2, lk.sx2, lk.sy2, lk.rho2, lk.amp2, ovf_cnt, ovf);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dloc = max(dloc, __shfl_xor_sync(~0u, dloc, o));
  if (lane == 0 && dloc) atomicMax(s_dmax, dloc);
  __syncthreads();
  // publish this source's counts and maximum diameter to every destination
  int* cnt_in = reinterpret_cast<int*>(X.smem + X.L.cnt_in_off) + b * 2 * C;
  float* dmax_in = reinterpret_cast<float*>(X.smem + X.L.dmax_in_off) + b * C;
  if (tid < 2 * C) {
    const int f = tid / C, d = tid - f * C;
    cl_st1(cl_map(cnt_in + f * C + k, (uint32_t)d), (uint32_t)X.cnt_out[tid]);
  } else if (tid >= 64 && tid < 64 + C) {
    cl_st1(cl_map(dmax_in + k, (uint32_t)(tid - 64)), *s_dmax);
  }
  __syncthreads();
  if (tid < 2 * C) X.cnt_out[tid] = 0;
}

// Per-pair kernel loop (pipelined over the cluster's pairs, one cluster
// barrier per pair):
//   A(first); barrier
//   for each pair k:  setup(k); B_1(k); C_1(k); B_2(k); A(k+1) -> buffer (k+1)&1;
//                     arrive; C_2(k); wait
// A(k+1) writes the buffer B(k-1) read: every destination finished B(k-1)
// before arriving at barrier k (after its A(k)); B(k+1) reads what A(k+1)
// wrote before barrier k+1. The store of frame 2 overlaps the barrier.
template <int PSF, bool SIMPLE, int WM>
__global__ void __launch_bounds__(kPairThreads, 2) pair_kernel(const BandParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ PairItem it;
  __shared__ unsigned s_dmax;
  __shared__ int s_M[2];
  __shared__ double s_ppp[2];
  constexpr int RW = RecW<SIMPLE>::kWords;
  constexpr int SEP = (PSF == kPsfPoint && WM > 0) ? 1 : 0;
  const int tid = threadIdx.x, lane = tid & 31;
  PairCtx<SIMPLE> X;
  X.C = P.cl_size;
  X.k = (int)cl_rank();
  X.smem = smem;
  X.L = pair_smem(P.cl_rows, P.pad_rows, P.AS, X.C, P.cl_cap, RW, 1);
  X.cnt_out = reinterpret_cast<int*>(smem + X.L.cnt_out_off);
  const int C = X.C, k = X.k;
  const int cid = (int)cl_id(), ncl = (int)cl_count();
  X.ovf_cnt = P.cl_ovf_cnt + (size_t)cid * 2 * C * 2;
  X.ovf = P.cl_ovf + (size_t)cid * 2 * C * 2 * P.n * RW;
  int* acc = reinterpret_cast<int*>(smem);
  const int r0 = k * P.cl_rows, r1 = min(P.H, r0 + P.cl_rows);
  for (int e = tid; e < X.L.acc_ints / 4; e += kPairThreads) reinterpret_cast<int4*>(acc)[e] = make_int4(0, 0, 0, 0);
  if (tid < 2 * C) X.cnt_out[tid] = 0;
  // every CTA of the cluster runs before anyone writes into its shared memory
  cl_arrive();
  cl_wait();
  const GenCfg& g = P.g;
  int pl = cid, b = 0;
  if (pl < P.pairs) pair_phase_a<SIMPLE>(P, X, pl, 0, s_M, s_ppp, &s_dmax);
  cl_arrive();
  cl_wait();
  for (; pl < P.pairs; pl += ncl, b ^= 1) {
    const int M = s_M[b];
    const int* cnt_in = reinterpret_cast<const int*>(smem + X.L.cnt_in_off) + b * 2 * C;
    const float* dmax_in = reinterpret_cast<const float*>(smem + X.L.dmax_in_off) + b * C;
    int* ovf_cnt_b = X.ovf_cnt + b * C * 2;
    const uint4* inbox = reinterpret_cast<const uint4*>(smem + X.L.inbox_off) + (size_t)b * X.L.buf_words;
    const uint4* ovf_k = X.ovf + ((size_t)b * C * 2 + (size_t)k * 2) * P.n * RW;
    // ---- setup (warp 0): maximum diameter -> side, inbox prefixes, shifts
    if (tid < 32) {
      float dm = lane < C ? dmax_in[lane] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dm = fmaxf(dm, __shfl_xor_sync(~0u, dm, o));
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const int c = lane < C ? min(cnt_in[f * C + lane], P.cl_cap) : 0;
        int x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(~0u, x, o);
          if (lane >= o) x += y;
        }
        if (lane < C) it.pre[f][lane + 1] = x;
        const int kin = __shfl_sync(~0u, x, 31);
        if (lane == 0) {
          it.pre[f][0] = 0;
          it.kin[f] = kin;
          it.K[f] = kin + __ldcg(ovf_cnt_b + k * 2 + f);
          // fixed-point shift: a pixel receives at most K contributions
          it.shift[f] = shift_for(max(1, it.K[f]), P.amp_bound);
          it.inv_scale[f] = 1.0f / (float)(1 << it.shift[f]);
        }
      }
      if (lane == 0) {
        // no active particle: the reference falls back to diameter_range[1] (pipeline.py:292)
        it.side = patch_side_exact(M > 0 ? (double)dm : g.d_hi, g.patch_mult);
        it.dmax = M > 0 ? dm : (float)g.d_hi;
        it.h = it.side >> 1;
        if (k == 0) {
          PairHdr hd{};
          hd.ppp = s_ppp[b];
          hd.M = M;
          hd.side = it.side;
          hd.dmax = it.dmax;
          write_stats(P, pl, hd);
        }
      }
    }
    __syncthreads();
    // ---- B_1, C_1, B_2: the accumulator holds one frame at a time
    pair_splat_frame<PSF, SEP, WM, SIMPLE>(P, inbox, acc, it, 0, r0, r1, ovf_k);
    __syncthreads();
    pair_store(P, acc, pl, 0, r0, r1 - r0, it.inv_scale[0]);
    __syncthreads();
    pair_splat_frame<PSF, SEP, WM, SIMPLE>(P, inbox, acc, it, 1, r0, r1, ovf_k + (size_t)P.n * RW);
    __syncthreads();
    if (tid < 2) ovf_cnt_b[k * 2 + tid] = 0;   // spill lists of buffer b consumed (self-cleaning)
    // ---- A(next pair) into the other buffer, while slower CTAs finish B(k)
    if (pl + ncl < P.pairs) pair_phase_a<SIMPLE>(P, X, pl + ncl, b ^ 1, s_M, s_ppp, &s_dmax);
    cl_arrive();
    // ---- C_2: store frame 2 while the barrier completes
    pair_store(P, acc, pl, 1, r0, r1 - r0, it.inv_scale[1]);
    __syncthreads();
    cl_wait();
  }
}

// Particle arrays of the pair law (sample_particles path): one thread per
// particle; the per-pair maximum diameter by atomicMax on the float bits.
__global__ void pair_particles_kernel(const BandParams P, pgb_particle_out O, unsigned* dmax_bits) {
  const int pl = blockIdx.y;
  const int gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= P.n) return;
  const GenCfg& g = P.g;
  const RngKey key = band_key(P, pl);
  const uint4 w0 = philox_rk(make_uint4(0u, key.pair, key.batch, kTagPair), g.rk);
  const double ppp = lerp_exact(g.ppp_lo, g.ppp_hi, u53_to_unit(w0.x, w0.y));
  double mm = rint(dmul(dmul(ppp, (double)g.H), (double)g.W));
  mm = fmin(fmax(mm, 0.0), (double)P.n);
  const int M = (int)mm;
  const bool active = gi < M;
  const float2* flow = P.flows + (size_t)((P.pair_base + pl) / P.pairs_per_field) * P.field_elems;
  PairPart pp;
  pair_particle(g, key, gi, flow, pp);
  if (!active) {
    // inactive capacity slots: I0 = 0, never rendered (particles.py:89)
    seed_look(g, key, gi, pp.sig, 0.f, pp.lk);
  } else {
    atomicMax(dmax_bits + pl, __float_as_uint(pp.d));
  }
  const Look& lk = pp.lk;
  const size_t o = (size_t)pl * P.n + gi;
  if (O.pos1) { O.pos1[2 * o] = (double)pp.xq1 * 0x1p-20; O.pos1[2 * o + 1] = (double)pp.yq1 * 0x1p-20; }
  if (O.pos2) { O.pos2[2 * o] = (double)pp.xq2 * 0x1p-20; O.pos2[2 * o + 1] = (double)pp.yq2 * 0x1p-20; }
  if (O.i0_1) O.i0_1[o] = lk.amp1;
  if (O.sx_1) O.sx_1[o] = pp.sig;
  if (O.sy_1) O.sy_1[o] = pp.sig;
  if (O.rho_1) O.rho_1[o] = lk.rho1;
  if (O.i0_2) O.i0_2[o] = lk.amp2;
  if (O.sx_2) O.sx_2[o] = lk.sx2;
  if (O.sy_2) O.sy_2[o] = lk.sy2;
  if (O.rho_2) O.rho_2[o] = lk.rho2;
  if (O.diameter) O.diameter[o] = pp.d;
  if (O.z1) O.z1[o] = lk.z1;
  if (O.active) O.active[o] = active ? 1 : 0;
  if (O.visible1) O.visible1[o] = (active && lk.vis1) ? 1 : 0;
  if (O.visible2) O.visible2[o] = (active && lk.vis2) ? 1 : 0;
}

__global__ void pair_stats_kernel(const BandParams P, const unsigned* dmax_bits) {
  const int pl = blockIdx.x * blockDim.x + threadIdx.x;
  if (pl >= P.pairs) return;
  const GenCfg& g = P.g;
  const RngKey key = band_key(P, pl);
  const uint4 w0 = philox_rk(make_uint4(0u, key.pair, key.batch, kTagPair), g.rk);
  const double ppp = lerp_exact(g.ppp_lo, g.ppp_hi, u53_to_unit(w0.x, w0.y));
  double mm = rint(dmul(dmul(ppp, (double)g.H), (double)g.W));
  mm = fmin(fmax(mm, 0.0), (double)P.n);
  PairHdr hd{};
  hd.ppp = ppp;
  hd.M = (int)mm;
  hd.dmax = hd.M > 0 ? __uint_as_float(dmax_bits[pl]) : (float)g.d_hi;
  hd.side = patch_side_exact(hd.M > 0 ? (double)hd.dmax : g.d_hi, g.patch_mult);
  write_stats(P, pl, hd);
}

}  // namespace pgb
