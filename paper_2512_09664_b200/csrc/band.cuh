// band.cuh -- the batched image-pair generator: prologue + band kernel.
//
// Replaces the body of Sampler._render_batch (reference pipeline.py:278-329):
// sample_particles / perturb_frame2 / advect / apply_hiding
// (particles.py:61-147), patch_side (raster.py:30-38, pipeline.py:291-294),
// splat (raster.py:108-126 -> _native.pyx:14-66), finalize (raster.py:154-161)
// and quantize_u16 (export.py:19-20).
//
// Design (B200-first):
//   * Stratified seeding. The M particle positions of a pair are iid uniform
//     over the image; we draw them as (cell counts, position inside the cell)
//     where the image is split into 2^sy x 2^sx equal-area seeding cells and
//     the counts are the histogram of M iid uniform cell labels -- exactly the
//     multinomial law of iid uniform positions. Particle g of the pair lives in
//     the cell whose prefix range holds g; all its other draws are keyed by g.
//     The per-pair maximum diameter (patch side, pipeline.py:292) is drawn
//     first (max of M uniforms ~ V^(1/M), carried by a uniform particle J; the
//     others are uniform below it) -- the same joint law, known up front.
//   * prologue_kernel (one CTA per pair): density, M, maximum diameter, the
//     cell histogram -> per-cell prefix; one CTA per flow field: max |u|,|v|.
//   * band_kernel (persistent, one item = one screen tile of one pair, both
//     frames): every CTA enumerates only the cells whose particles can reach
//     its tile (tile + patch half-width + the field's max displacement),
//     regenerates those particles from their counters, advects them and splats
//     them straight into a shared-memory fixed-point accumulator (int32,
//     2^-s units: integer adds are associative -> bit-identical results for
//     any schedule), then runs the fused epilogue (offset + Philox noise +
//     clamp, optional uint16) with 128-bit streaming stores. No inter-CTA
//     communication, no global intermediates: HBM traffic = the images.
#pragma once
#include "fused.cuh"

namespace pgb {

// Timing probes (build with -DPGB_TRACE only; scripts/trace.py reads them):
// globaltimer stamps per CTA, slot = blockIdx.x * kTraceSlots + event.
#ifdef PGB_TRACE
constexpr int kTraceSlots = 40;   // 0-15 events, 16 + 3k.. item k phases (k < 6), 34-38 part/window events, 39 smid
__device__ unsigned long long g_trace[2048 * kTraceSlots];
__device__ __forceinline__ void trace_stamp(int ev) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  if (blockIdx.x < 2048) g_trace[blockIdx.x * kTraceSlots + ev] = t;
}
#define PGB_STAMP(ev) do { if (threadIdx.x == 0) trace_stamp(ev); } while (0)
// first-item stamps (stager lane 0): a shared flag, not a read-back of
// g_trace (a global load would add an L2 round trip to the stamped interval)
__shared__ int g_trace_first;
__shared__ int g_trace_item;   // items rendered so far (worker thread 0)
__device__ __forceinline__ void trace_item(int phase) {
  if (threadIdx.x == 0 && g_trace_item < 6) trace_stamp(16 + 3 * g_trace_item + phase);
}
#else
#define PGB_STAMP(ev) do { } while (0)
#endif

#ifdef PGB_BAND_MAXREG
#define PGB_BAND_BOUNDS __maxnreg__(PGB_BAND_MAXREG)
#else
#ifndef PGB_BAND_MINB
#define PGB_BAND_MINB 2
#endif
#define PGB_BAND_BOUNDS __launch_bounds__(kBandBlock, PGB_BAND_MINB)   // 2 CTAs x 288 threads per SM
#endif
#ifndef PGB_WORKER_WARPS
#define PGB_WORKER_WARPS 8
#endif
constexpr int kBandThreads = 32 * PGB_WORKER_WARPS;
constexpr int kBandWarps = kBandThreads / 32;
constexpr int kBandBlock = kBandThreads + 32;   // + one staging warp
constexpr int kMaxCellBits = 14;
constexpr int kMaxUnpredWM = 12;   // largest unpredicated (separable) splat window
constexpr int kSortClasses = 5;    // sorted splat window classes: 4, 6, 8, 10, 12
constexpr int kSortMinW = 7;       // items whose window bound reaches this use the sorted splat
constexpr int kLaneWM = kSortMinW - 1;   // largest per-lane unpredicated window (code size: the
                                         // kernel holds one unrolled particle loop per window)
constexpr int kVarSorted = 100;    // ItemCfg::var of the sorted splat

struct __align__(16) PairHdr {
  double ppp;      // realised seeding density
  double m;        // continuous maximum diameter uniform (0 when M == 0)
  int M;           // active particles
  int J;           // particle carrying the maximum
  int qmax;        // 23-bit quantised maximum
  int side;        // patch side of the pair
  float dmax;      // maximum diameter
  int cmax;        // max particles in one seeding cell
  int pad0, pad1;
};

struct BandParams {
  int H, W;
  int TH, TW, AS, tiles_y, tiles_x, tiles;
  // items: (pair, tile) for item < split_base; the remaining tiles are split
  // into split_s row parts each (the last, partial round of the static
  // schedule spread over all CTAs); total_items = split_base + rem * split_s
  long long split_base, total_items;
  int split_s;
  int pad_rows;                // zero rows after the frame-2 accumulator (unpredicated splat windows)
  int rec_bytes;               // SortShared region ahead of the accumulators (sorted splat), else 0
  int pro_smem;                // shared bytes the pair prologue may use (prologue kernel / band accumulators)
  int sy, sx;                  // seeding cells: 2^sy rows x 2^sx columns
  double inv_ch, inv_cw;       // 2^sy / H, 2^sx / W (cells per pixel)
  int n, pairs;
  long long pair_base;
  uint32_t batch_lo;
  int psf, out_mode;
  float bg_offset, noise_std;
  float amp_bound;             // upper bound of any particle amplitude
  GenCfg g;
  const float2* flows;
  int pairs_per_field, num_fields;
  long long field_elems;
  float2* fbound;              // [num_fields] (max |u|, max |v|)
  int* prefix;                 // [pairs][2^(sy+sx) + 1] particle prefix per cell
  unsigned short* cell_of;     // [pairs][cof_stride(n)] seeding cell of every active particle
  PairHdr* hdr;                // [pairs]
  int* pair_ready;             // [pairs] prologue done (in-kernel prologue), else null
  int* fb_done;                // [num_fields] finished bound chunks, else null
  long long npro;              // prologue tickets ahead of the band items: flow-bound chunks, histogram
                               // parts (pro_parts > 1), pair prologues, particle -> cell windows (fill_wins)
  int pro_parts;               // histogram parts per pair on other CTAs (1: the prologue draws all labels)
  int* part_counts;            // [pairs][pro_parts][2^(sy+sx)] partial cell histograms (pro_parts > 1)
  int* part_done;              // [pairs] finished histogram parts
  int fill_win, fill_wins;     // particle -> cell windows per pair on other CTAs (0: the prologue fills)
  int* pre_ready;              // [pairs] header + prefix published (fill windows wait on it)
  int* fill_done;              // [pairs] finished particle -> cell windows
  int4* zero_head;             // the other control head: zeroed here for the next launch (or null)
  int zero_head_n;
  int field_lo, field_cnt;     // flow fields read by this pair range
  void* out[2];
  long long out_pair_elems;
  double* st_ppp;
  int* st_M;
  int* st_side;
  float* st_dmax;
  int* ticket;
};

// Per-pair cell prefix stride (ints): ncell + 1 entries, padded for 16-byte rows.
__host__ __device__ __forceinline__ size_t pre_stride(int ncell) { return (size_t)ncell + 4; }
// Per-pair particle -> cell stride (u16): n padded to 16-byte rows.
__host__ __device__ __forceinline__ size_t cof_stride(int n) { return ((size_t)n + 7) & ~(size_t)7; }

// ----------------------------------------------------------------------------
// Seeding pieces shared by the band kernel and the particle-array kernel
// ----------------------------------------------------------------------------
__device__ __forceinline__ RngKey band_key(const BandParams& P, int pl) {
  return RngKey{P.g.k0, P.g.k1, (uint32_t)(P.pair_base + pl), P.batch_lo};
}

// 23-bit diameter quantile of particle g: the maximum qmax sits on particle J,
// the others are uniform on [0, qmax] (floor(w (qmax + 1) / 2^32)).
__device__ __forceinline__ int diam_q(const PairHdr& hd, int g, uint32_t wz) {
  return g == hd.J ? hd.qmax : (int)__umulhi(wz, (uint32_t)hd.qmax + 1u);
}

__device__ __forceinline__ float q_to_unit(int q) { return ((float)q + 0.5f) * 0x1p-23f; }

// Advection of a fixed-point point: bilinear, edge-clamped (flowfield.py:207-232)
// in float32, then the new anchor/fraction (see fused.cuh gen_particle).
__device__ __forceinline__ void advect_fixed(const GenCfg& g, const float2* __restrict__ flow,
                                             uint32_t X, uint32_t Y, int ax, float fx, int ay,
                                             float fy, int& ax2, float& fx2, int& ay2, float& fy2) {
  int cx, cy;
  float tx, ty;
  fixed_cell(X, g.W, cx, tx);
  fixed_cell(Y, g.H, cy, ty);
  const int cx1 = cx + 1 < g.W ? cx + 1 : g.W - 1;
  const int cy1 = cy + 1 < g.H ? cy + 1 : g.H - 1;
  const float2 q00 = __ldg(flow + (size_t)cy * g.W + cx);
  const float2 q01 = __ldg(flow + (size_t)cy * g.W + cx1);
  const float2 q10 = __ldg(flow + (size_t)cy1 * g.W + cx);
  const float2 q11 = __ldg(flow + (size_t)cy1 * g.W + cx1);
  const float u = bilerp(q00.x, q01.x, q10.x, q11.x, tx, ty);
  const float v = bilerp(q00.y, q01.y, q10.y, q11.y, tx, ty);
  advect_anchor(X, ax, u, ax2, fx2);
  advect_anchor(Y, ay, v, ay2, fy2);
}

// Appearance of both frames (particles.py:61-126 + laser sheet), given the
// active particle's diameter and i0. Keyed by the particle index g.
struct Look {
  float amp1, amp2, sx2, sy2, rho1, rho2, z1;
  bool vis1, vis2;
};

__device__ __forceinline__ void seed_look(const GenCfg& g, const RngKey& key, int gi, float sig,
                                          float i0, Look& lk) {
  float rho = g.rho_lo, z1 = 0.f;
  bool vis1 = true, vis2 = true;
  if (g.need_b) {
    const uint4 b = philox_rk(make_uint4((uint32_t)gi, key.pair, key.batch, kTagParticleB), g.rk);
    rho = lerpf_exact(g.rho_lo, g.rho_span, unit23(b.x));
    vis1 = (uint64_t)b.y >= g.hide_thr;   // apply_hiding (particles.py:139-147)
    vis2 = (uint64_t)b.z >= g.hide_thr;
    z1 = lerpf_exact(g.z_lo, g.z_span, unit23(b.w));
  }
  float sx2 = sig, sy2 = sig, i02 = i0, rho2 = rho;
  if (g.need_perturb) {
    // perturb_frame2 (particles.py:104-126)
    const uint4 c = philox_rk(make_uint4((uint32_t)gi, key.pair, key.batch, kTagPerturb), g.rk);
    const float2 n01 = box_muller(c.x, c.y);
    const float2 n23 = box_muller(c.z, c.w);
    if (g.f2_sigma_std > 0.f) {
      sx2 = fmaxf(__fadd_rn(sig, __fmul_rn(g.f2_sigma_std, n01.x)), 1e-3f);
      sy2 = fmaxf(__fadd_rn(sig, __fmul_rn(g.f2_sigma_std, n01.y)), 1e-3f);
    }
    if (g.f2_i0_std > 0.f) {
      const float t = fminf(fmaxf(__fadd_rn(i0, __fmul_rn(g.f2_i0_std, n23.x)), 0.f), 1.f);
      i02 = i0 == 0.f ? 0.f : t;
    }
    if (g.f2_rho_std > 0.f) {
      const float lim = 0.999f;
      rho2 = fminf(fmaxf(__fadd_rn(rho, __fmul_rn(g.f2_rho_std, n23.y)), -lim), lim);
    }
  }
  float amp1 = i0, amp2 = i02;
  if (g.laser) {
    amp1 *= laser_profile(g, z1);
    amp2 *= laser_profile(g, z1 + g.w);
  }
  lk.amp1 = amp1; lk.amp2 = amp2; lk.sx2 = sx2; lk.sy2 = sy2;
  lk.rho1 = rho; lk.rho2 = rho2; lk.z1 = z1; lk.vis1 = vis1; lk.vis2 = vis2;
}

// Full particle (both frames) for the particle-array API (sample_particles).
__device__ __forceinline__ void seed_particle(const BandParams& P, const PairHdr& hd, int pl, int gi,
                                              int cy, int cx, const float2* __restrict__ flow,
                                              Particle& pt) {
  const GenCfg& g = P.g;
  const RngKey key = band_key(P, pl);
  const uint4 a = philox_rk(make_uint4((uint32_t)gi, key.pair, key.batch, kTagParticleA), g.rk);
  const bool active = gi < hd.M;
  uint32_t X, Y;
  float d;
  if (active) {
    X = cell_coord((uint32_t)cx, a.x, g.W, P.sx);
    Y = cell_coord((uint32_t)cy, a.y, g.H, P.sy);
    d = lerpf_exact(g.d_lo, g.d_span, q_to_unit(diam_q(hd, gi, a.z)));
  } else {
    // inactive capacity slots: full-image uniforms, never rendered
    X = cell_coord(0u, a.x, g.W, 0);
    Y = cell_coord(0u, a.y, g.H, 0);
    d = lerpf_exact(g.d_lo, g.d_span, unit23(a.z));
  }
  const float i0 = lerpf_exact(g.i0_lo, g.i0_span, unit23(a.w));
  const float i0f = active ? i0 : 0.f;
  const float sig = __fmul_rn(d, g.inv_ratio);
  Look lk;
  seed_look(g, key, gi, sig, i0f, lk);
  Frame& f1 = pt.fr[0];
  Frame& f2 = pt.fr[1];
  fixed_anchor(X, f1.ax, f1.fx);
  fixed_anchor(Y, f1.ay, f1.fy);
  advect_fixed(g, flow, X, Y, f1.ax, f1.fx, f1.ay, f1.fy, f2.ax, f2.fx, f2.ay, f2.fy);
  f1.amp = lk.amp1; f1.sx = sig; f1.sy = sig; f1.rho = lk.rho1;
  f2.amp = lk.amp2; f2.sx = lk.sx2; f2.sy = lk.sy2; f2.rho = lk.rho2;
  f1.on = active && lk.vis1 && lk.amp1 > 0.f;
  f2.on = active && lk.vis2 && lk.amp2 > 0.f;
  pt.diam = d;
  pt.z1 = lk.z1;
  pt.active = active;
  pt.vis1 = lk.vis1 && active;
  pt.vis2 = lk.vis2 && active;
}

// ----------------------------------------------------------------------------
// Prologue: one CTA per pair (+ one per flow field)
// ----------------------------------------------------------------------------
constexpr int kPrologueThreads = 512;
constexpr int kFieldBlocks = 16;   // work chunks per flow field for the displacement bound

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_b(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Flow bound, one of kFieldBlocks chunks of field f (whole block): max |u|,
// max |v| by atomicMax on the bits of non-negative floats (non-finite values
// -> unbounded); the chunk counter fb_done[f] releases the bound.
template <int NT>
__device__ __forceinline__ void field_bound_chunk(const BandParams& P, int f, int part) {
  const int tid = threadIdx.x, lane = tid & 31;
  const float2* fl = P.flows + (size_t)f * P.field_elems;
  float mu = 0.f, mv = 0.f;
  auto take = [&](const float2 v) {
    const float au = fabsf(v.x), av = fabsf(v.y);
    mu = au <= 3.0e38f ? fmaxf(mu, au) : INFINITY;
    mv = av <= 3.0e38f ? fmaxf(mv, av) : INFINITY;
  };
  // the chunk is a contiguous range of the field read as 16-byte pairs of
  // nodes, eight loads in flight per thread (the bound gates the first band
  // items: latency, not bandwidth, matters)
  const long long n = P.field_elems;
  const long long per = ((n + kFieldBlocks - 1) / kFieldBlocks + 1) & ~1LL;
  const long long lo = min(n, (long long)part * per), hi = min(n, lo + per);
  const float4* f4 = reinterpret_cast<const float4*>(fl + lo);   // lo even
  const bool vec = (reinterpret_cast<uintptr_t>(fl) & 15) == 0;
  const long long n4 = vec ? (hi - lo) >> 1 : 0;
  if (!vec)
    for (long long e = lo + tid; e < hi; e += NT) take(__ldg(fl + e));
  for (long long q0 = 0; q0 < n4; q0 += 8LL * NT) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long q = q0 + (long long)k * NT + tid;
      v[k] = q < n4 ? __ldg(f4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      take(make_float2(v[k].x, v[k].y));
      take(make_float2(v[k].z, v[k].w));
    }
  }
  if (vec && ((hi - lo) & 1) && tid == 0) take(__ldg(fl + hi - 1));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mu = fmaxf(mu, __shfl_xor_sync(~0u, mu, o));
    mv = fmaxf(mv, __shfl_xor_sync(~0u, mv, o));
  }
  if (lane == 0) {
    unsigned* b = reinterpret_cast<unsigned*>(P.fbound + f);
    atomicMax(b, __float_as_uint(mu));
    atomicMax(b + 1, __float_as_uint(mv));
  }
  __syncthreads();
  if (tid == 0 && P.fb_done) {
    __threadfence();
    atomicAdd(P.fb_done + f, 1);
  }
}

__device__ __forceinline__ void write_stats(const BandParams& P, int pl, const PairHdr& hd) {
  if (P.st_ppp) P.st_ppp[pl] = hd.ppp;
  if (P.st_M) P.st_M[pl] = hd.M;
  if (P.st_side) P.st_side[pl] = hd.side;
  if (P.st_dmax) P.st_dmax[pl] = hd.dmax;
}

// Named barrier of the scan warps (every warp of the block but the last).
template <int NTS>
__device__ __forceinline__ void scan_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NTS) : "memory");
}

// The last warp's share of the prologue: the pair's maximum diameter. The max
// of M uniforms is V^(1/M) (a serial float64 chain), carried by particle J.
__device__ __forceinline__ void pair_max_diameter(const GenCfg& g, const RngKey& key, int M, PairHdr& hd) {
  hd.M = M;
  hd.m = 0.0;
  hd.J = 0;
  hd.qmax = 0;
  float dmax = (float)g.d_hi;
  if (M > 0) {
    const uint4 v = philox_rk(make_uint4(1u, key.pair, key.batch, kTagPair), g.rk);
    const double V = u53_to_unit(v.x, v.y);
    hd.m = rexp(ddiv(rlog(V), (double)M));
    hd.J = (int)__umul64hi(((uint64_t)v.w << 32) | v.z, (uint64_t)M);
    const int q = (int)floor(hd.m * 8388608.0);
    hd.qmax = q < 0x7fffff ? q : 0x7fffff;
    dmax = lerpf_exact(g.d_lo, g.d_span, q_to_unit(hd.qmax));
  }
  hd.dmax = dmax;
  // no active particle: the reference falls back to diameter_range[1] (pipeline.py:292)
  hd.side = patch_side_exact(M > 0 ? (double)dmax : g.d_hi, g.patch_mult);
}

// Per-pair prologue (whole block of NT threads; `bins` = the shared scratch of
// smem_bytes bytes): density, M, maximum diameter, the cell histogram -> per-cell
// prefix and the particle -> cell array; pair_ready[pl] releases them.
// Latency-bound (one pair per CTA at the start of every launch), so the last
// warp draws the maximum diameter (a serial float64 chain) while the others
// histogram and scan, synchronised by a named barrier of their own.
// Cell histogram of labels 4q .. 4q+3 (< M) for Philox calls q in
// [q_lo, q_hi) (4 labels per call; up to four calls in flight per thread), by
// the NTS scan threads, with shared-memory atomics into bins.
template <int NTS>
__device__ __forceinline__ void hist_labels(const GenCfg& g, const RngKey& key, int M, int L, int* bins,
                                            int q_lo, int q_hi) {
  const int tid = threadIdx.x;
  const int nq = (M + 3) >> 2;   // the last call, q = nq - 1, may hold labels >= M
  const int q_full = min(q_hi, nq - 1);
  int q = q_lo + tid;
  // full groups, unconditional atomics
  for (; q + 3 * NTS < q_full; q += 4 * NTS) {
    const uint4 a = philox_rk(make_uint4((uint32_t)q, key.pair, key.batch, kTagCell), g.rk);
    const uint4 b = philox_rk(make_uint4((uint32_t)(q + NTS), key.pair, key.batch, kTagCell), g.rk);
    const uint4 c = philox_rk(make_uint4((uint32_t)(q + 2 * NTS), key.pair, key.batch, kTagCell), g.rk);
    const uint4 d = philox_rk(make_uint4((uint32_t)(q + 3 * NTS), key.pair, key.batch, kTagCell), g.rk);
    const uint32_t ws[16] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w, d.x, d.y, d.z, d.w};
#pragma unroll
    for (int k = 0; k < 16; ++k) atomicAdd(&bins[L ? (ws[k] >> (32 - L)) : 0], 1);
  }
  // the rest (< 4 calls per thread, up to the partial last call): one group,
  // its calls in flight together, checked atomics
  if (q < q_hi) {
    uint4 w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      w[k] = philox_rk(make_uint4((uint32_t)(q + k * NTS), key.pair, key.batch, kTagCell), g.rk);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int qk = q + k * NTS;
      const uint32_t ws[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (qk < q_hi && 4 * qk + e < M) atomicAdd(&bins[L ? (ws[e] >> (32 - L)) : 0], 1);
    }
  }
}

// Particle -> cell (counting-sort order: particles of cell c are
// pre[c] .. pre[c+1]-1) for slots [s_lo, s_hi) in windows of `win` slots
// staged in shared memory behind the prefix (bins); the NTS scan threads.
// one_win: the slots were zeroed and the run starts marked during the prefix
// pass (the whole pair in one window).
template <int NTS>
__device__ __forceinline__ void fill_slots(const int* bins, int ncell, int M, int s_lo, int s_hi, int win,
                                           bool one_win, unsigned short* scof, unsigned short* cof) {
  constexpr int NS = NTS / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int4* s4 = reinterpret_cast<int4*>(scof);
  const int M8 = s_hi;
  // particle -> cell (counting-sort order: particles of cell c are
  // pre[c] .. pre[c+1]-1), per window of slots: mark the first slot of every
  // cell starting in the window with the cell id, inclusive max-scan (carry
  // in: the cell holding the window's first slot), 16-byte stores
  __shared__ int wcar[128];                     // per-chunk carries of one window
  auto max8 = [](const int4 w) {
    const int a = max(max(w.x & 0xffff, (int)((unsigned)w.x >> 16)), max(w.y & 0xffff, (int)((unsigned)w.y >> 16)));
    const int b = max(max(w.z & 0xffff, (int)((unsigned)w.z >> 16)), max(w.w & 0xffff, (int)((unsigned)w.w >> 16)));
    return max(a, b);
  };
  // dense cells (>= 2 particles per cell on average, e.g. C3's 6.4): every
  // cell writes its run into the window directly (no scans); sparse cells
  // (C2's 0.5) mark run starts and max-scan
  const bool dense = M >= 2 * ncell;
  for (int s0 = s_lo; s0 < M8; s0 += win) {
    const int s1 = min(M8, s0 + win);
    const int n4 = (s1 - s0) >> 3;               // int4 groups of 8 slots
    if (!one_win && !dense)
      for (int q = tid; q < n4; q += NTS) s4[q] = make_int4(0, 0, 0, 0);
    // the cell holding slot s0: last c with bins[c] <= s0 (and a non-empty run)
    int clo = 0;
    if (s0 > 0) {
      int lo = 0, hi = ncell - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (bins[mid] <= s0) lo = mid;
        else hi = mid - 1;
      }
      clo = lo;   // bins is non-decreasing and bins[ncell] = M > s0: cell clo holds slot s0
    }
    if (dense) {
      int chi = ncell - 1;   // last cell with a slot in the window
      if (s1 < M) {
        int lo = clo, hi = ncell - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (bins[mid] < s1) lo = mid;
          else hi = mid - 1;
        }
        chi = lo;
      }
      for (int cb = clo + warp * 32; cb <= chi; cb += NTS) {   // warp-uniform trip count
        const int c = cb + lane;
        int j0 = 0, n = 0;
        if (c <= chi) {
          j0 = max(bins[c], s0);
          n = min(bins[c + 1], s1) - j0;
        }
        const int nmax = __reduce_max_sync(~0u, n);
        for (int k = 0; k < nmax; ++k)
          if (k < n) scof[j0 + k - s0] = (unsigned short)c;
      }
      if (tid < 8 && M + tid < s1) scof[M + tid - s0] = 0;   // padding slots of the last window
      scan_sync<NTS>();
      const int4* src = reinterpret_cast<const int4*>(scof);
      int4* dst = reinterpret_cast<int4*>(cof + s0);
      for (int q = tid; q < n4; q += NTS) dst[q] = src[q];
      if (s1 < M8) scan_sync<NTS>();
      continue;
    }
    if (!one_win) {
      // cells starting inside the window: (clo, chi], chi = last c with bins[c] < s1
      int chi = ncell - 1;
      if (s1 < M) {
        int lo = clo, hi = ncell - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (bins[mid] < s1) lo = mid;
          else hi = mid - 1;
        }
        chi = lo;
      }
      scan_sync<NTS>();
#pragma unroll 4
      for (int c = clo + tid; c <= chi; c += NTS) {
        const int b = bins[c];
        if (b >= s0 && b < bins[c + 1]) scof[b - s0] = (unsigned short)c;
      }
      scan_sync<NTS>();
    }
    // chunk maxima (256 slots = one warp layer of int4s per chunk)
    const int nch = (n4 + 31) >> 5;
    for (int ch = warp; ch < nch; ch += NS) {
      const int q = (ch << 5) + lane;
      int mx = q < n4 ? max8(s4[q]) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(~0u, mx, o));
      if (lane == 0) wcar[ch] = mx;
    }
    scan_sync<NTS>();
    if (warp == 0) {
      int carry = clo;
      for (int c0 = 0; c0 < nch; c0 += 32) {
        const int c = c0 + lane;
        int m = c < nch ? wcar[c] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(~0u, m, o);
          if (lane >= o) m = max(m, y);
        }
        const int up = __shfl_up_sync(~0u, m, 1);
        const int ex = max(carry, lane ? up : 0);
        if (c < nch) wcar[c] = ex;
        carry = max(carry, __shfl_sync(~0u, m, 31));
      }
    }
    scan_sync<NTS>();
    int4* c4 = reinterpret_cast<int4*>(cof + s0);
    for (int ch = warp; ch < nch; ch += NS) {
      const int q = (ch << 5) + lane;
      int4 w4 = make_int4(0, 0, 0, 0);
      if (q < n4) w4 = s4[q];
      int m = max8(w4);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(~0u, m, o);
        if (lane >= o) m = max(m, y);
      }
      const int prev = __shfl_up_sync(~0u, m, 1);
      int r = lane > 0 ? max(wcar[ch], prev) : wcar[ch];
      int lo, hi, o0, o1, o2, o3;
      lo = r = max(r, w4.x & 0xffff); hi = r = max(r, (int)((unsigned)w4.x >> 16)); o0 = lo | (hi << 16);
      lo = r = max(r, w4.y & 0xffff); hi = r = max(r, (int)((unsigned)w4.y >> 16)); o1 = lo | (hi << 16);
      lo = r = max(r, w4.z & 0xffff); hi = r = max(r, (int)((unsigned)w4.z >> 16)); o2 = lo | (hi << 16);
      lo = r = max(r, w4.w & 0xffff); hi = r = max(r, (int)((unsigned)w4.w >> 16)); o3 = lo | (hi << 16);
      if (q < n4) c4[q] = make_int4(o0, o1, o2, o3);
    }
    if (s1 < M8) scan_sync<NTS>();
  }
}

template <int NT>
__device__ __forceinline__ void pair_prologue(const BandParams& P, int pl, int* bins, int smem_bytes) {
  constexpr int NW = NT / 32;
  constexpr int NS = NW - 1;          // scan warps
  constexpr int NTS = NS * 32;
  static_assert(NS >= 1 && NS <= 32, "prologue warps");
  __shared__ PairHdr shd;
  __shared__ int ctot[32];            // chunk bases (<= 32 chunks of 512 cells)
  __shared__ int wmx[NS];
  __shared__ int stot, scm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int L = P.sy + P.sx;
  const int ncell = 1 << L;
  const int nc4 = ncell < 4 ? 4 : ncell;
  const RngKey key = band_key(P, pl);
  const GenCfg& g = P.g;
  PGB_STAMP(2);
  // seeding density and active count (particles.py:73-83), computed by every
  // thread (identical values)
  const uint4 w0 = philox_rk(make_uint4(0u, key.pair, key.batch, kTagPair), g.rk);
  const double ppp = lerp_exact(g.ppp_lo, g.ppp_hi, u53_to_unit(w0.x, w0.y));
  double mm = rint(dmul(dmul(ppp, (double)g.H), (double)g.W));
  mm = fmin(fmax(mm, 0.0), (double)P.n);
  const int M = (int)mm;
  int* pre = P.prefix + (size_t)pl * pre_stride(ncell);
  unsigned short* cof = P.cell_of + (size_t)pl * cof_stride(P.n);
  // particle -> cell slots staged in shared memory behind the prefix, in
  // windows of `win` slots (one window: marked during the prefix pass)
  const int soff = ((nc4 + 4) & ~3) * 4;
  unsigned short* scof = reinterpret_cast<unsigned short*>(reinterpret_cast<char*>(bins) + soff);
  int4* s4 = reinterpret_cast<int4*>(scof);
  const int win = max(8, min(128 * 256, ((smem_bytes - soff) / 2) & ~7));   // slots per window (plans leave >= 8)
  const int M8 = (M + 7) & ~7;
  // one window, sparse cells: run starts marked during the prefix pass, then
  // a max-scan; dense cells (>= 2 particles per cell: C2's 128 full-width cell
  // rows hold ~31 each) write their runs directly (fill_slots)
  const bool one_win = M8 <= win && M < 2 * ncell;
  if (warp == NS) {
    if (lane == 0) {
      PairHdr hd;
      pair_max_diameter(g, key, M, hd);
      hd.ppp = ppp;
      shd = hd;
#ifdef PGB_TRACE
      trace_stamp(14);
#endif
    }
  } else {
    int4* bins4 = reinterpret_cast<int4*>(bins);
    const int nq4 = nc4 >> 2;                    // int4 groups of cells
    for (int i = tid; i < nq4; i += NTS) bins4[i] = make_int4(0, 0, 0, 0);
    if (one_win)
      for (int q = tid; q < (M8 >> 3); q += NTS) s4[q] = make_int4(0, 0, 0, 0);
    scan_sync<NTS>();
    if (P.pro_parts > 1) {
      // the histogram was drawn in parts by other CTAs (earlier tickets): sum them
      if (tid == 0) {
        int ns = 32;
        while (ld_acquire_b(P.part_done + pl) < P.pro_parts) { __nanosleep(ns); ns = min(ns * 2, 256); }
      }
      scan_sync<NTS>();
      // (all loads of four rows x up to four parts in flight: a dependent
      // loop over parts was one L2 round trip per row, ~10 us at C3)
      const int4* pc = reinterpret_cast<const int4*>(P.part_counts + (size_t)pl * P.pro_parts * ncell);
      const int K = P.pro_parts;
      for (int i0 = tid; i0 < nq4; i0 += 4 * NTS) {
        int4 v[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = i0 + j * NTS;
            v[j][k] = (i < nq4 && k < K) ? __ldcg(pc + (size_t)k * (ncell >> 2) + i) : make_int4(0, 0, 0, 0);
          }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + j * NTS;
          const int4 t = make_int4(v[j][0].x + v[j][1].x + v[j][2].x + v[j][3].x,
                                   v[j][0].y + v[j][1].y + v[j][2].y + v[j][3].y,
                                   v[j][0].z + v[j][1].z + v[j][2].z + v[j][3].z,
                                   v[j][0].w + v[j][1].w + v[j][2].w + v[j][3].w);
          if (i < nq4) bins4[i] = t;
        }
      }
    } else {
      hist_labels<NTS>(g, key, M, L, bins, 0, (M + 3) >> 2);
    }

    scan_sync<NTS>();
    PGB_STAMP(3);
    // Cell counts -> exclusive prefix (in place + global) and the maximum cell
    // count. Warps own 512-cell chunks (four 128-cell layers, lanes reading
    // consecutive int4s); chunk totals combined by warp 0.
    const int nchunk = (nq4 + 127) >> 7;
    int cm = 0;
    for (int ch = warp; ch < nchunk; ch += NS) {
      int tot = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int q = (ch << 7) + (j << 5) + lane;
        const int4 v = q < nq4 ? bins4[q] : make_int4(0, 0, 0, 0);
        tot += v.x + v.y + v.z + v.w;
        cm = max(cm, max(max(v.x, v.y), max(v.z, v.w)));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(~0u, tot, o);
      if (lane == 0) ctot[ch] = tot;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cm = max(cm, __shfl_xor_sync(~0u, cm, o));
    if (lane == 0) wmx[warp] = cm;
    scan_sync<NTS>();
    if (warp == 0) {
      const int t = lane < nchunk ? ctot[lane] : 0;
      int v = t;
      int m = lane < NS ? wmx[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(~0u, v, o);
        if (lane >= o) v += y;
        m = max(m, __shfl_xor_sync(~0u, m, o));
      }
      if (lane < nchunk) ctot[lane] = v - t;   // exclusive chunk bases
      if (lane == 31) stot = v;
      if (lane == 0) scm = m;
    }
    scan_sync<NTS>();
    PGB_STAMP(4);
    // in-chunk prefix: the four layers' warp scans interleaved (independent),
    // then chained by their totals
    int4* pre4 = reinterpret_cast<int4*>(pre);
    for (int ch = warp; ch < nchunk; ch += NS) {
      int4 v[4];
      int sv[4], inc[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int q = (ch << 7) + (j << 5) + lane;
        v[j] = q < nq4 ? bins4[q] : make_int4(0, 0, 0, 0);
        sv[j] = v[j].x + v[j].y + v[j].z + v[j].w;
        inc[j] = sv[j];
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int y = __shfl_up_sync(~0u, inc[j], o);
          if (lane >= o) inc[j] += y;
        }
      }
      int run = ctot[ch];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int q = (ch << 7) + (j << 5) + lane;
        const int b0 = run + inc[j] - sv[j];
        const int4 o4 = make_int4(b0, b0 + v[j].x, b0 + v[j].x + v[j].y, b0 + v[j].x + v[j].y + v[j].z);
        if (q < nq4) {
          bins4[q] = o4;   // exclusive prefix, in place (entries >= ncell: the total)
          const int i = q << 2;
          if (i + 4 <= ncell) {
            pre4[q] = o4;
          } else {
            const int oo[4] = {o4.x, o4.y, o4.z, o4.w};
            for (int k = 0; i + k < ncell; ++k) pre[i + k] = oo[k];
          }
          if (one_win) {
            // mark the first slot of every non-empty cell with the cell id
            if (v[j].x) scof[o4.x] = (unsigned short)i;
            if (v[j].y) scof[o4.y] = (unsigned short)(i + 1);
            if (v[j].z) scof[o4.z] = (unsigned short)(i + 2);
            if (v[j].w) scof[o4.w] = (unsigned short)(i + 3);
          }
        }
        run += __shfl_sync(~0u, inc[j], 31);
      }
    }
    if (tid == 0) {
      bins[ncell] = stot;
      pre[ncell] = stot;
    }
    scan_sync<NTS>();
    PGB_STAMP(5);
    if (P.fill_wins == 0) fill_slots<NTS>(bins, ncell, M, 0, M8, win, one_win, scof, cof);
  }
  __syncthreads();   // the maximum-diameter warp joins
  PGB_STAMP(6);
  if (tid == 0) {
    PairHdr hd = shd;
    hd.cmax = scm;
    P.hdr[pl] = hd;
    write_stats(P, pl, hd);
    // The block's prefix / particle -> cell writes are ordered before this
    // thread by the barrier above, its own header write by program order; a
    // release store is cumulative over both (the bar.sync + st.release.gpu
    // publish pattern), so no separate fence. Particle -> cell windows on
    // other CTAs release the pair when there are any.
    if (P.pair_ready) st_release(P.fill_wins ? P.pre_ready + pl : P.pair_ready + pl, 1);
  }
  PGB_STAMP(7);
}

// Histogram part k of pair pl (pro_parts > 1; whole block, the scan warps
// draw): labels of Philox calls [k nq / K, (k+1) nq / K) into shared memory,
// then to part_counts; part_done[pl] counts the finished parts.
template <int NT>
__device__ __forceinline__ void pair_hist_part(const BandParams& P, int pl, int k, int* bins) {
  constexpr int NTS = (NT / 32 - 1) * 32;
  const int tid = threadIdx.x;
  const int L = P.sy + P.sx, ncell = 1 << L;
  const RngKey key = band_key(P, pl);
  const GenCfg& g = P.g;
  const uint4 w0 = philox_rk(make_uint4(0u, key.pair, key.batch, kTagPair), g.rk);
  const double ppp = lerp_exact(g.ppp_lo, g.ppp_hi, u53_to_unit(w0.x, w0.y));
  double mm = rint(dmul(dmul(ppp, (double)g.H), (double)g.W));
  mm = fmin(fmax(mm, 0.0), (double)P.n);
  const int M = (int)mm;
  const int nq = (M + 3) >> 2;
  const int K = P.pro_parts;
  int4* bins4 = reinterpret_cast<int4*>(bins);
  PGB_STAMP(34);
  for (int i = tid; i < (ncell >> 2); i += NT) bins4[i] = make_int4(0, 0, 0, 0);
  __syncthreads();
  if (tid < NTS) hist_labels<NTS>(g, key, M, L, bins, (int)((long long)nq * k / K), (int)((long long)nq * (k + 1) / K));
  __syncthreads();
  PGB_STAMP(35);
  int4* dst = reinterpret_cast<int4*>(P.part_counts + ((size_t)pl * K + k) * ncell);
  for (int i = tid; i < (ncell >> 2); i += NT) dst[i] = bins4[i];
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    atomicAdd(P.part_done + pl, 1);
  }
  PGB_STAMP(36);
}

// Particle -> cell window w of pair pl (fill_wins > 0; whole block, the scan
// warps fill): waits for the pair's prefix, stages it in shared memory, fills
// the window; the last window of the pair releases it.
template <int NT>
__device__ __forceinline__ void pair_fill_window(const BandParams& P, int pl, int w, int* bins) {
  constexpr int NTS = (NT / 32 - 1) * 32;
  __shared__ int sM;
  const int tid = threadIdx.x;
  const int L = P.sy + P.sx, ncell = 1 << L, nc4 = ncell < 4 ? 4 : ncell;
  if (tid == 0) {
    int ns = 32;
    while (ld_acquire_b(P.pre_ready + pl) == 0) { __nanosleep(ns); ns = min(ns * 2, 256); }
    sM = __ldcg(&P.hdr[pl].M);
  }
  __syncthreads();
  PGB_STAMP(37);
  const int M = sM, M8 = (M + 7) & ~7;
  const int s0 = w * P.fill_win, s1 = min(M8, s0 + P.fill_win);
  if (s0 < s1) {
    // the prefix row (ncell + 4 ints, 16-byte aligned) as int4s, eight loads
    // in flight per thread (one dependent L2 round trip per int was ~10 us
    // of the C3 start-up chain)
    const int* pre = P.prefix + (size_t)pl * pre_stride(ncell);
    if ((ncell & 3) == 0) {
      // loads first, then the shared stores: interleaved, the compiler cannot
      // move a load above the previous (possibly aliasing) store, and every
      // row costs a full L2 round trip (measured 9 us per C3 window)
      const int4* pre4 = reinterpret_cast<const int4*>(pre);
      int4* b4 = reinterpret_cast<int4*>(bins);
      const int n4 = (int)(pre_stride(ncell) >> 2);
      for (int i0 = tid; i0 < n4; i0 += 8 * NT) {
        int4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = i0 + j * NT;
          v[j] = i < n4 ? __ldcg(pre4 + i) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = i0 + j * NT;
          if (i < n4) b4[i] = v[j];
        }
      }
    } else {
      for (int i = tid; i <= ncell; i += NT) bins[i] = __ldcg(pre + i);
    }
    __syncthreads();
    const int soff = ((nc4 + 4) & ~3) * 4;
    unsigned short* scof = reinterpret_cast<unsigned short*>(reinterpret_cast<char*>(bins) + soff);
    unsigned short* cof = P.cell_of + (size_t)pl * cof_stride(P.n);
    if (tid < NTS) fill_slots<NTS>(bins, ncell, M, s0, s1, P.fill_win, false, scof, cof);
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(P.fill_done + pl, 1) == P.fill_wins - 1) {
      __threadfence();
      st_release(P.pair_ready + pl, 1);
    }
  }
  PGB_STAMP(38);
}

// Standalone prologue (sample_particles path): one CTA per pair + kFieldBlocks
// per flow field.
__global__ void __launch_bounds__(kPrologueThreads) prologue_kernel(const BandParams P) {
  extern __shared__ int bins[];
  PGB_STAMP(0);
  if (blockIdx.x >= P.pairs) {
    const int fb = blockIdx.x - P.pairs;
    field_bound_chunk<kPrologueThreads>(P, fb / kFieldBlocks, fb % kFieldBlocks);
    PGB_STAMP(12);
    return;
  }
  pair_prologue<kPrologueThreads>(P, blockIdx.x, bins, P.pro_smem);
  PGB_STAMP(12);
}

// ----------------------------------------------------------------------------
// Band kernel
// ----------------------------------------------------------------------------
// Per-item parameters (warp 0 computes them for the next item while the
// block finishes the current one; double-buffered).
constexpr int kMaxSeg = 128;   // particle segments (cell rows) per enumeration pass
constexpr int kStageSlots = 2; // staged item slots (current + next)

struct ItemCfg {
  int pl, r0, r1, c0, c1;
  int cy0, cy1, cx0, cx1;
  int h, wt, shift, field, sep;
  int var;                 // particle-loop variant: 16 * sep + WM (0 = dynamic windows)
  float2 fb;               // the field's displacement bound (max |u|, max |v|)
  int kind;                // kItemBand or kItemEnd
  long long item;          // band item index
  PairHdr hd;
};
enum { kItemBand = 0, kItemEnd = 2 };

struct __align__(16) BandShared {
  int wsum[kBandWarps];
  long long ticket0;                 // prologue / first band ticket of this CTA
  long long ticket_next;             // the following ticket, taken while a prologue item runs

  int nseg[kStageSlots];             // segments of the staged pass
  int rows_left[kStageSlots];        // cell rows not yet staged (rare multi-pass items)
  ItemCfg ic[kStageSlots];
  int seg_start[kStageSlots][kMaxSeg];       // first particle index of each segment
  int seg_off[kStageSlots][kMaxSeg + 1];     // exclusive prefix of segment lengths
};

__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Tight window of one particle-frame (anchor offsets clipped to +-h), then
// clipped to the tile [r0, r1) x [c0, c1). Returns false when empty.
__device__ __forceinline__ bool tile_window(int ax, int ay, float fx, float fy, float R, int h, int r0,
                                            int r1, int c0, int c1, int& rlo, int& clo, int& nr,
                                            int& nc) {
  const int jlo = max(-h, (int)ceilf(__fsub_rn(fx, R)));
  const int jhi = min(h, (int)floorf(__fadd_rn(fx, R)));
  const int ilo = max(-h, (int)ceilf(__fsub_rn(fy, R)));
  const int ihi = min(h, (int)floorf(__fadd_rn(fy, R)));
  rlo = max(ay + ilo, r0);
  const int rhi = min(ay + ihi, r1 - 1);
  clo = max(ax + jlo, c0);
  const int chi = min(ax + jhi, c1 - 1);
  nr = rhi - rlo + 1;
  nc = chi - clo + 1;
  return nr > 0 && nc > 0;
}

// Point PSF, one particle-frame (one lane): WM = compile-time bound of the
// window side (columns and rows fully unrolled, predicated), 0 = dynamic.
// value * 2^s = exp2(Ls - A dx^2 - B dx dy - C dy^2), rounded to an integer.
template <int WM>
__device__ __forceinline__ void splat_point(int* __restrict__ acc, int AS, int ax, int ay, float fx,
                                            float fy, float amp, float sx, float sy, float rho, int h,
                                            int r0, int r1, int c0, int c1, int shift) {
  const float R = __fmul_rn(fmaxf(sx, sy), kTightR);
  int rlo, clo, nr, nc;
  if (!tile_window(ax, ay, fx, fy, R, h, r0, r1, c0, c1, rlo, clo, nr, nc)) return;
  const float dx0 = (float)(clo - ax) - fx;
  const float dy0 = (float)(rlo - ay) - fy;
  int* base = acc + (rlo - r0) * AS + (clo - c0);
  const float isx = rcp_approx(sx), isy = rcp_approx(sy);
  const float iq = rcp_approx(1.0f - rho * rho);
  const float A = (0.5f * kLog2e) * iq * isx * isx;
  const float C = (0.5f * kLog2e) * iq * isy * isy;
  const float B = -kLog2e * rho * iq * isx * isy;
  const float Ls = lg2_approx(amp) + (float)shift;
  if (WM > 0) {
    // pixels beyond the bound lie outside the tight radius (they round to 0)
    nr = min(nr, WM);
    nc = min(nc, WM);
    float ct[WM > 0 ? WM : 1], bx[WM > 0 ? WM : 1];
#pragma unroll
    for (int j = 0; j < WM; ++j) {
      const float dx = dx0 + (float)j;
      ct[j] = fmaf(-A * dx, dx, Ls);
      bx[j] = B * dx;
    }
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      if (i < nr) {
        const float dy = dy0 + (float)i;
        const float rt = -C * dy * dy;
        int* row = base + i * AS;
#pragma unroll
        for (int j = 0; j < WM; ++j)
          if (j < nc) atomicAdd(row + j, round_small(ex2_approx(fmaf(-bx[j], dy, ct[j] + rt))));
      }
    }
  } else {
    for (int i = 0; i < nr; ++i) {
      const float dy = dy0 + (float)i;
      const float bt = B * dy;
      const float rt = fmaf(-C * dy, dy, Ls);
      int* row = base + i * AS;
      for (int j = 0; j < nc; ++j) {
        const float dx = dx0 + (float)j;
        atomicAdd(row + j, round_small(ex2_approx(fmaf(-dx, fmaf(A, dx, bt), rt))));
      }
    }
  }
}

// Pixel-area mean of Eq. (1) (oracle/render.py render_erf), one particle-frame.
__device__ __forceinline__ void splat_erf(int* __restrict__ acc, int AS, int ax, int ay, float fx,
                                          float fy, float amp, float sx, float sy, float rho, int h,
                                          int r0, int r1, int c0, int c1, float scale) {
  const float R = __fadd_rn(__fmul_rn(fmaxf(sx, sy), kTightR), 0.5f);
  int rlo, clo, nr, nc;
  if (!tile_window(ax, ay, fx, fy, R, h, r0, r1, c0, c1, rlo, clo, nr, nc)) return;
  const float dx0 = (float)(clo - ax) - fx;
  const float dy0 = (float)(rlo - ay) - fy;
  int* base = acc + (rlo - r0) * AS + (clo - c0);
  const float k = 1.2533141373155001f;  // sqrt(pi/2)
  const float sc = sx * sqrtf(fmaxf(1.0f - rho * rho, 0.f));
  const bool sep = rho == 0.f;
  const float Lm = (sep ? amp * (k * sx) * (k * sy) : amp * (k * sc)) * scale;
  const float rA = 0.70710678118654752f / sc;
  const float rB = 0.70710678118654752f / sy;
  const float rC = sep ? 0.f : rho * sx / sy;
  for (int i = 0; i < nr; ++i) {
    const float dy = dy0 + (float)i;
    const float ey = sep ? erff((dy + 0.5f) * rB) - erff((dy - 0.5f) * rB) : 0.f;
    for (int j = 0; j < nc; ++j) {
      const float dx = dx0 + (float)j;
      float val;
      if (sep) {
        val = (erff((dx + 0.5f) * rA) - erff((dx - 0.5f) * rA)) * ey;
      } else {
        float s = 0.f;
#pragma unroll
        for (int gq = 0; gq < kGLPoints; ++gq) {
          const float yy = dy + kGLx[gq];
          const float mu = rC * yy;
          const float gy = __expf(-yy * yy * (rB * rB));
          const float hi = erff((dx + 0.5f - mu) * rA);
          const float lo = erff((dx - 0.5f - mu) * rA);
          s = fmaf(kGLw[gq] * gy, hi - lo, s);
        }
        val = s;
      }
      const int qv = __float2int_rn(val * Lm);
      if (qv) atomicAdd(base + i * AS + j, qv);
    }
  }
}

// Unpredicated separable point-PSF windows (WM = compile-time window bound,
// 1..kLaneWM; uncorrelated particles, one particle-frame per lane).
// Every particle-frame adds all WM x WM slots; slots outside its clipped
// window add exactly 0 (their factor is 0), so no per-slot branch is needed. Slots past the tile's last row / column land on
// the next row or on the zero padding after the frame-2 accumulator
// (pad_rows >= WM - 1 rows), always with value 0.
template <int WM>
__device__ __forceinline__ void splat_sep_u(int* __restrict__ acc, int AS, int ax, int ay, float fx,
                                            float fy, float amp, float sx, float sy, int h, int r0,
                                            int r1, int c0, int c1, int shift) {
  const float R = __fmul_rn(fmaxf(sx, sy), kTightR);
  int rlo, clo, nr, nc;
  if (!tile_window(ax, ay, fx, fy, R, h, r0, r1, c0, c1, rlo, clo, nr, nc)) return;
  const float dx0 = (float)(clo - ax) - fx;
  const float dy0 = (float)(rlo - ay) - fy;
  int* base = acc + (rlo - r0) * AS + (clo - c0);
  const float isx = rcp_approx(sx), isy = rcp_approx(sy);
  const float A = (0.5f * kLog2e) * isx * isx;
  const float C = (0.5f * kLog2e) * isy * isy;
  const float Ls = lg2_approx(amp) + (float)shift;
  float X[WM];
#pragma unroll
  for (int j = 0; j < WM; ++j) {
    const float dx = dx0 + (float)j;
    const float xv = ex2_approx(fmaf(-A * dx, dx, Ls));
    X[j] = j < nc ? xv : 0.f;
  }
  if constexpr (WM <= 7) {
    float Y[WM];
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      const float dy = dy0 + (float)i;
      const float yv = ex2_approx(-C * dy * dy);
      Y[i] = i < nr ? yv : 0.f;
    }
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      int* row = base + i * AS;
#pragma unroll
      for (int j = 0; j < WM; ++j)
        atomicAdd(row + j, __float_as_int(fmaf(X[j], Y[i], 12582912.0f)) - 0x4B400000);
    }
  } else {
    // large windows: rows in a loop (one exponential per row), columns unrolled
#pragma unroll 1
    for (int i = 0; i < WM; ++i) {
      const float dy = dy0 + (float)i;
      const float yv = ex2_approx(-C * dy * dy);
      const float Y = i < nr ? yv : 0.f;
      int* row = base + i * AS;
#pragma unroll
      for (int j = 0; j < WM; ++j)
        atomicAdd(row + j, __float_as_int(fmaf(X[j], Y, 12582912.0f)) - 0x4B400000);
    }
  }
}

// One particle-frame, variant fixed per item: SEP (rho == 0 everywhere),
// WM (1..kLaneWM unpredicated separable windows; 0 = dynamic loops).
template <int PSF, int SEP, int WM>
__device__ __forceinline__ void splat_v(int* acc, int AS, int ax, int ay, float fx, float fy, float amp,
                                        float sx, float sy, float rho, int h, int r0, int r1, int c0,
                                        int c1, int shift, float scale) {
  if constexpr (PSF == kPsfErf) {
    splat_erf(acc, AS, ax, ay, fx, fy, amp, sx, sy, rho, h, r0, r1, c0, c1, scale);
  } else if constexpr (WM == 0) {
    splat_point<0>(acc, AS, ax, ay, fx, fy, amp, sx, sy, rho, h, r0, r1, c0, c1, shift);
  } else {
    static_assert(SEP != 0, "unpredicated windows are instantiated for uncorrelated particles only");
    splat_sep_u<WM>(acc, AS, ax, ay, fx, fy, amp, sx, sy, h, r0, r1, c0, c1, shift);
  }
}

// Epilogue: one output quad (4 pixels) of frame f. (float)a is exact below
// 2^24 and correctly rounded above (the accumulator stays < 2^31).
// Round keys held in registers for the noise epilogue (the store loop would
// otherwise reload the 20 key words from the constant bank every iteration).
__device__ __forceinline__ uint32_t in_reg(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ PhiloxKeys keys_in_regs(const PhiloxKeys& K) {
  PhiloxKeys R;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    R.k0[r] = in_reg(K.k0[r]);
    R.k1[r] = in_reg(K.k1[r]);
  }
  return R;
}

template <int OUT, bool NOISE>
__device__ __forceinline__ void band_store_quad(const BandParams& P, int4 a, char* dst, uint32_t pix,
                                                int f, uint32_t gpair, float inv_scale,
                                                const PhiloxKeys& K) {
  float4 v = make_float4((float)a.x, (float)a.y, (float)a.z, (float)a.w);
  if (OUT == kOutRaw) {
    v.x *= inv_scale; v.y *= inv_scale; v.z *= inv_scale; v.w *= inv_scale;
    __stcs(reinterpret_cast<float4*>(dst), v);
    return;
  }
  const float bg = P.bg_offset;
  if (NOISE) {
    // finalize_px(acc * 2^-s, ...) as FFMA.SAT(acc, 2^-s, offset + std * n)
    const float sd = P.noise_std;
    const float4 nz = noise4_rk(K, gpair, P.batch_lo, (uint32_t)f + 1, pix >> 2);
    v.x = __saturatef(fmaf(v.x, inv_scale, fmaf(sd, nz.x, bg)));
    v.y = __saturatef(fmaf(v.y, inv_scale, fmaf(sd, nz.y, bg)));
    v.z = __saturatef(fmaf(v.z, inv_scale, fmaf(sd, nz.z, bg)));
    v.w = __saturatef(fmaf(v.w, inv_scale, fmaf(sd, nz.w, bg)));
  } else {
    v.x = __saturatef(fmaf(v.x, inv_scale, bg));   // clip(raw + offset, 0, 1): FFMA.SAT
    v.y = __saturatef(fmaf(v.y, inv_scale, bg));
    v.z = __saturatef(fmaf(v.z, inv_scale, bg));
    v.w = __saturatef(fmaf(v.w, inv_scale, bg));
  }
  if (OUT == kOutF32) {
    __stcs(reinterpret_cast<float4*>(dst), v);
  } else {
    ushort4 u = make_ushort4(quant_u16(v.x), quant_u16(v.y), quant_u16(v.z), quant_u16(v.w));
    __stcs(reinterpret_cast<ushort4*>(dst), u);
  }
}

// Store one frame of the tile and zero its accumulator (quad path: tile
// columns, image width and tile origin multiples of 4). Each thread walks its
// quads with incremental row/column/pointer updates (no per-quad division or
// 64-bit index arithmetic).
template <int OUT, bool NOISE>
__device__ __forceinline__ void band_store_vec(const BandParams& P, int* __restrict__ acc, int pl, int f, int r0,
                               int nr, int c0, int nc, float inv_scale) {
  constexpr int ESZ = OUT == kOutU16 ? 2 : 4;
  const uint32_t gpair = (uint32_t)(P.pair_base + pl);
  const int qpr = nc >> 2;
  if (nr <= 0 || qpr <= 0) return;
  const int tid = threadIdx.x;
  int row = tid / qpr, cq = tid - (tid / qpr) * qpr;
  const int drow = kBandThreads / qpr, dcq = kBandThreads - drow * qpr;
  const int W = P.W, AS = P.AS;
  uint32_t pix = (uint32_t)((r0 + row) * W + c0 + cq * 4);
  int ao = row * AS + cq * 4;
  char* dst = static_cast<char*>(P.out[f]) + ((size_t)pl * (size_t)P.out_pair_elems + pix) * ESZ;
  const uint32_t dpix = (uint32_t)(drow * W + dcq * 4);
  const int dao = drow * AS + dcq * 4;
  const uint32_t wrap_pix = (uint32_t)(W - qpr * 4);
  const int wrap_ao = AS - qpr * 4;
  const PhiloxKeys K = NOISE ? keys_in_regs(P.g.rk) : P.g.rk;
  if (dcq == 0) {
    // qpr divides the block: every thread keeps its column quad
    const size_t ddst = (size_t)dpix * ESZ;
    for (; row < nr; row += drow, pix += dpix, ao += dao, dst += ddst) {
      int4* ap = reinterpret_cast<int4*>(acc + ao);
      const int4 a = *ap;
      *ap = make_int4(0, 0, 0, 0);
      band_store_quad<OUT, NOISE>(P, a, dst, pix, f, gpair, inv_scale, K);
    }
    return;
  }
  while (row < nr) {
    int4* ap = reinterpret_cast<int4*>(acc + ao);
    const int4 a = *ap;
    *ap = make_int4(0, 0, 0, 0);
    band_store_quad<OUT, NOISE>(P, a, dst, pix, f, gpair, inv_scale, K);
    row += drow;
    cq += dcq;
    pix += dpix;
    ao += dao;
    dst += (size_t)dpix * ESZ;
    if (cq >= qpr) {
      cq -= qpr;
      ++row;
      pix += wrap_pix;
      ao += wrap_ao;
      dst += (size_t)wrap_pix * ESZ;
    }
  }
}

// Full-width tile (c0 == 0, nc == W == AS): the tile is one contiguous run of
// quads in shared memory and in the output; each thread strides the quads.
template <int OUT, bool NOISE>
__device__ __forceinline__ void band_store_lin(const BandParams& P, int* __restrict__ acc, int pl, int f,
                                               int r0, int nr, float inv_scale, int t = threadIdx.x,
                                               int nt = kBandThreads) {
  constexpr int ESZ = OUT == kOutU16 ? 2 : 4;
  const uint32_t gpair = (uint32_t)(P.pair_base + pl);
  const int nq = (nr * P.W) >> 2;
  const uint32_t pix0 = (uint32_t)(r0 * P.W);
  char* dst = static_cast<char*>(P.out[f]) + ((size_t)pl * (size_t)P.out_pair_elems + pix0) * ESZ;
  int4* ap = reinterpret_cast<int4*>(acc);
  if constexpr (NOISE) {
    const PhiloxKeys K = keys_in_regs(P.g.rk);
#pragma unroll 2
    for (int q = t; q < nq; q += nt) {
      const int4 a = ap[q];
      ap[q] = make_int4(0, 0, 0, 0);
      band_store_quad<OUT, NOISE>(P, a, dst + (size_t)q * 4 * ESZ, pix0 + 4u * q, f, gpair, inv_scale, K);
    }
  } else {
#pragma unroll 4
    for (int q = t; q < nq; q += nt) {
      const int4 a = ap[q];
      ap[q] = make_int4(0, 0, 0, 0);
      band_store_quad<OUT, NOISE>(P, a, dst + (size_t)q * 4 * ESZ, pix0 + 4u * q, f, gpair, inv_scale, P.g.rk);
    }
  }
}

__device__ __forceinline__ void band_store_scalar(const BandParams& P, int* __restrict__ acc, int pl, int f, int r0,
                                  int nr, int c0, int nc, float inv_scale) {
  const uint32_t gpair = (uint32_t)(P.pair_base + pl);
  const size_t pair_off = (size_t)pl * (size_t)P.out_pair_elems;
  const int mode = P.out_mode;
  const float bg = P.bg_offset, sd = P.noise_std;
  const int total = nr * nc;
  for (int e = threadIdx.x; e < total; e += kBandThreads) {
    const int row = e / nc;
    const int col = e - row * nc;
    int* ap = acc + row * P.AS + col;
    float v = (float)*ap * inv_scale;
    *ap = 0;
    const size_t p = (size_t)(r0 + row) * P.W + (size_t)(c0 + col);
    if (mode == kOutRaw) {
      static_cast<float*>(P.out[f])[pair_off + p] = v;
    } else {
      float nzv = 0.f;
      if (sd > 0.f) {
        const float4 nz = noise4_rk(P.g.rk, gpair, P.batch_lo, (uint32_t)f + 1, (uint32_t)(p >> 2));
        const int jn = (int)(p & 3);
        nzv = jn == 0 ? nz.x : (jn == 1 ? nz.y : (jn == 2 ? nz.z : nz.w));
      }
      v = finalize_px(v, bg, sd, nzv);
      if (mode == kOutF32) static_cast<float*>(P.out[f])[pair_off + p] = v;
      else static_cast<uint16_t*>(P.out[f])[pair_off + p] = quant_u16(v);
    }
  }
}

// Full-width tiles are stored by the whole block (the staging warp joins: it
// has staged the next item by then); other tiles by the worker warps.
__device__ __forceinline__ bool store_is_lin(const BandParams& P, int c0, int nc) {
  return ((nc & 3) == 0) && ((P.W & 3) == 0) && c0 == 0 && nc == P.W && P.AS == P.W;
}

__device__ __forceinline__ void band_store(const BandParams& P, int* acc, int pl, int f, int r0, int nr, int c0, int nc,
                           float inv_scale) {
  const bool vec = ((nc & 3) == 0) && ((P.W & 3) == 0) && ((c0 & 3) == 0);
  const bool noise = P.noise_std > 0.f;
  if (store_is_lin(P, c0, nc)) {
    const int t = threadIdx.x, nt = kBandBlock;
    switch (P.out_mode) {
      case kOutRaw: band_store_lin<kOutRaw, false>(P, acc, pl, f, r0, nr, inv_scale, t, nt); return;
      case kOutF32:
        if (noise) band_store_lin<kOutF32, true>(P, acc, pl, f, r0, nr, inv_scale, t, nt);
        else band_store_lin<kOutF32, false>(P, acc, pl, f, r0, nr, inv_scale, t, nt);
        return;
      default:
        if (noise) band_store_lin<kOutU16, true>(P, acc, pl, f, r0, nr, inv_scale, t, nt);
        else band_store_lin<kOutU16, false>(P, acc, pl, f, r0, nr, inv_scale, t, nt);
        return;
    }
  }
  if (threadIdx.x >= kBandThreads) return;
  if (vec) {
    switch (P.out_mode) {
      case kOutRaw: band_store_vec<kOutRaw, false>(P, acc, pl, f, r0, nr, c0, nc, inv_scale); return;
      case kOutF32:
        if (noise) band_store_vec<kOutF32, true>(P, acc, pl, f, r0, nr, c0, nc, inv_scale);
        else band_store_vec<kOutF32, false>(P, acc, pl, f, r0, nr, c0, nc, inv_scale);
        return;
      default:
        if (noise) band_store_vec<kOutU16, true>(P, acc, pl, f, r0, nr, c0, nc, inv_scale);
        else band_store_vec<kOutU16, false>(P, acc, pl, f, r0, nr, c0, nc, inv_scale);
        return;
    }
  }
  band_store_scalar(P, acc, pl, f, r0, nr, c0, nc, inv_scale);
}


// Range of seeding cells [lo, hi] whose span [k*s, (k+1)*s) meets [a, b)
// (inv = 1/s; the callers' bounds carry >= 1/2 px of slack, far above the
// float rounding of a*inv (< 1e-3 px for frames below 2^13 px), so no
// division and no FP64 on the staging path: FP64 made the first item's
// parameters a ~1 us dependent chain at every launch start).
__device__ __forceinline__ void cell_range(float a, float b, float inv, int n, int& lo, int& hi) {
  const float fa = floorf(fmaxf(a, 0.f) * inv);
  const float fb = floorf(fminf(b * inv, (float)n));
  lo = (int)fminf(fa, (float)(n - 1));
  hi = (int)fminf(fmaxf(fb, 0.f), (float)(n - 1));
}

// Fixed-point shift without a division: the largest e <= kAccShift with
// cnt * (amp 2^e + 1/2) <= 2^31 (the contributions of `cnt` particles of
// amplitude <= amp, each rounded up by at most 1/2, fit an int32). Float
// arithmetic rounded upwards (products and sums, plus a 2^-20 margin): it
// may give one bit less than the exact bound at the boundary, never more.
__device__ __forceinline__ int shift_for_fast(int cnt, float amp) {
  const float ca = __fmul_ru(__fmul_ru(__int2float_ru(cnt), amp), 1.f + 0x1p-20f);
  if (!(ca > 0.f)) return kAccShift;
  int e = min(kAccShift, 31 - ilogbf(ca));
  while (e > 0 && __fadd_ru(ldexpf(ca, e), __fmul_ru(0.5f, __int2float_ru(cnt))) > 2147483648.f) --e;
  return e;
}

// The parameters only the staging path reads, loaded once by the stager's
// lane 0 at kernel entry (overlapping the first ticket's atomic): otherwise
// their constant-cache misses are serial latency in the first item's staging.
__device__ __forceinline__ void touch_stage_params(const BandParams& P) {
  asm volatile("" ::"l"(P.split_base), "r"(P.split_s), "r"(P.tiles), "r"(P.tiles_x), "r"(P.TH), "r"(P.TW),
               "r"(P.sy), "r"(P.sx), "d"(P.inv_ch), "d"(P.inv_cw), "f"(P.amp_bound), "r"(P.pairs_per_field),
               "l"(P.pair_base), "l"(P.hdr), "l"(P.fbound), "l"(P.pair_ready));
  asm volatile("" ::"l"(P.fb_done), "l"(P.prefix), "f"(P.g.f2_sigma_std), "d"(P.g.d_hi), "f"(P.g.inv_ratio),
               "f"(P.g.rho_lo), "f"(P.g.rho_span), "f"(P.g.f2_rho_std), "r"(P.psf), "r"(P.rec_bytes),
               "r"(P.pad_rows), "l"(P.total_items), "l"(P.npro), "r"(P.g.H));
}

// Item parameters (lane 0 of warp 0): tile, the cells whose particles can reach
// it, the fixed-point shift and the window bound.
__device__ __forceinline__ void item_finish(const BandParams& P, ItemCfg& ic);

__device__ __forceinline__ void item_setup(const BandParams& P, long long item, ItemCfg& ic) {
  const GenCfg& g = P.g;
  long long ti = item;
  int sub = 0, nsub = 1;
  if (item >= P.split_base) {
    const long long j = item - P.split_base;
    ti = P.split_base + j / P.split_s;
    sub = (int)(j % P.split_s);
    nsub = P.split_s;
  }
  const int pl = (int)(ti / P.tiles);
  const int t = (int)(ti - (long long)pl * P.tiles);
  const int ty = t / P.tiles_x, tx = t - ty * P.tiles_x;
  ic.pl = pl;
  ic.r0 = ty * P.TH;
  ic.r1 = min(ic.r0 + P.TH, g.H);
  if (nsub > 1) {
    const int ph = (ic.r1 - ic.r0 + nsub - 1) / nsub;
    const int a = min(ic.r1, ic.r0 + sub * ph);
    ic.r1 = min(ic.r1, a + ph);
    ic.r0 = a;   // may be empty (r0 == r1): no particles, no store
  }
  ic.c0 = tx * P.TW;
  ic.c1 = min(ic.c0 + P.TW, g.W);
  ic.field = (int)((P.pair_base + pl) / P.pairs_per_field);
  if (P.pair_ready) {
    // produced inside this launch by other CTAs (earlier tickets); both flags
    // polled together (one L2 round trip when they are already set)
    int ns = 32;
    for (;;) {
      const int a = ld_acquire_b(P.pair_ready + pl);
      const int b = ld_acquire_b(P.fb_done + ic.field);
      if (a != 0 && b >= kFieldBlocks) break;
      __nanosleep(ns);
      ns = min(ns * 2, 256);
    }
  }
#ifdef PGB_TRACE
  if (g_trace_first == 0) trace_stamp(10);
#endif
  {
    // header and field bound loaded together
    const int4* src = reinterpret_cast<const int4*>(P.hdr + pl);
    int4 t[sizeof(PairHdr) / 16];
#pragma unroll
    for (int k = 0; k < (int)(sizeof(PairHdr) / 16); ++k) t[k] = __ldcg(src + k);
    ic.fb = __ldcg(P.fbound + ic.field);
    int4* dst = reinterpret_cast<int4*>(&ic.hd);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(PairHdr) / 16); ++k) dst[k] = t[k];
  }
#ifdef PGB_TRACE
  // (conditioned on the loaded data so the stamp waits for the loads)
  if (g_trace_first == 0 && ic.hd.M >= -1 && ic.fb.x > -1.f) trace_stamp(11);
#endif
  item_finish(P, ic);
#ifdef PGB_TRACE
  if (g_trace_first == 0 && ic.shift >= 0 && ic.cy1 >= -1 && ic.cx1 >= -1 && ic.var >= 0) {
    trace_stamp(15);
    g_trace_first = 1;
  }
#endif
}

// Item parameters from the tile, the pair header (ic.hd) and the field bound:
// the cells whose particles can reach the tile, the fixed-point shift and the
// window bound / particle-loop variant.
__device__ __forceinline__ void item_finish(const BandParams& P, ItemCfg& ic) {
  const GenCfg& g = P.g;
  const int CY = 1 << P.sy, CX = 1 << P.sx;
  const int h = ic.hd.side >> 1;
  ic.h = h;
  const float2 fb = ic.fb;
  // frame-1 positions that can reach the tile in either frame: anchors within
  // h of the tile (frame 1), or within h + 1 + max|v| (frame 2: the anchor
  // moves by floor(f + v + 1/2), |f| <= 1/2); slack covers float rounding.
  const float vy = __fmaf_ru(fb.y, 1.f + 1e-6f, 1e-6f);
  const float vx = __fmaf_ru(fb.x, 1.f + 1e-6f, 1e-6f);
  const float inv_ch = (float)P.inv_ch, inv_cw = (float)P.inv_cw;
  cell_range((float)(ic.r0 - h) - 1.5f - vy, (float)(ic.r1 + h) + 0.5f + vy, inv_ch, CY, ic.cy0, ic.cy1);
  cell_range((float)(ic.c0 - h) - 1.5f - vx, (float)(ic.c1 + h) + 0.5f + vx, inv_cw, CX, ic.cx0, ic.cx1);
  // fixed-point shift: contributions per pixel <= cmax * (cells one pixel's
  // source box can meet), amplitude <= amp_bound (the 1e-4 keeps the floor
  // of an exact quotient from rounding down; a larger bound is only safer)
  const int by = (int)floorf(__fmaf_ru(2.f * vy + (float)(2 * h + 3), inv_ch, 1e-4f)) + 2;
  const int bx = (int)floorf(__fmaf_ru(2.f * vx + (float)(2 * h + 3), inv_cw, 1e-4f)) + 2;
  const long long cov = min((long long)ic.hd.M, (long long)ic.hd.cmax * min(by, CY) * min(bx, CX));
  ic.shift = shift_for_fast(max(1, (int)cov), P.amp_bound);
  // window side bound: floor(2 R_max) + 1 columns/rows, R_max from the largest
  // sigma (frame-2 sigma jitter is unbounded -> patch side)
  int wt = 2 * h + 1;
  if (P.psf == kPsfPoint && !(g.f2_sigma_std > 0.f)) {
    const float smax = __fmul_rn(ic.hd.M > 0 ? ic.hd.dmax : (float)g.d_hi, g.inv_ratio);
    const float Rm = __fmul_rn(smax, kTightR);
    wt = min(wt, (int)floorf(2.0f * Rm) + 1);
  }
  ic.wt = max(1, wt);
  // uncorrelated particles (rho == 0 in both frames): separable splat
  ic.sep = (g.rho_lo == 0.f && g.rho_span == 0.f && !(g.f2_rho_std > 0.f)) ? 1 : 0;
  // unpredicated windows for uncorrelated particles only: the correlated
  // variant (splat_point_u) showed tiling-dependent 1-ulp differences in the
  // stress test (scripts/stress.py); correlated particles use the dynamic loops
  // (per-lane unpredicated windows up to kLaneWM; larger separable windows
  // take the bank-sorted splat, or the dynamic loops when PGB_NO_SORT)
  const int wm = (P.psf == kPsfPoint && ic.sep && ic.wt <= kLaneWM && ic.wt - 1 <= P.pad_rows) ? ic.wt : 0;
  ic.var = (P.psf == kPsfPoint ? 16 * ic.sep : 0) + wm;
  // large separable windows: bank-sorted splat (plans with a record region)
  // (records need no padding rows: make_rec keeps windows inside the frame)
  if (P.rec_bytes && P.psf == kPsfPoint && ic.sep && ic.wt >= kSortMinW && ic.wt <= kMaxUnpredWM)
    ic.var = kVarSorted;
}

// Warp 0: next item's parameters + particle segments (one per cell row of the
// cell rectangle; a full-width rectangle is one contiguous segment).
__device__ __forceinline__ void item_stage(const BandParams& P, long long item, BandShared* sh, int b,
                                           int row_lo) {
  const int lane = threadIdx.x & 31;
  if (lane == 0 && row_lo == -1) item_setup(P, item, sh->ic[b]);
  __syncwarp();
  const ItemCfg& ic = sh->ic[b];
  const int CX = 1 << P.sx;
  const int* pre = P.prefix + (size_t)ic.pl * pre_stride((1 << P.sy) * CX);
  auto ldp = [&](size_t i) { return __ldcg(pre + i); };
  const bool full = ic.cx0 == 0 && ic.cx1 == CX - 1;
  const int y0 = row_lo < 0 ? ic.cy0 : row_lo;
  const int nrows = ic.cy1 - y0 + 1;
  const int nseg = ic.r0 >= ic.r1 ? 0 : (full ? 1 : min(nrows, kMaxSeg));   // empty split part: nothing
  int base = 0;
  for (int s0 = 0; s0 < nseg; s0 += 32) {
    const int sidx = s0 + lane;
    int st = 0, len = 0;
    if (sidx < nseg) {
      if (full) {
        st = ldp((size_t)ic.cy0 << P.sx);
        len = ldp((size_t)(ic.cy1 + 1) << P.sx) - st;
      } else {
        const int cy = y0 + sidx;
        st = ldp(((size_t)cy << P.sx) + ic.cx0);
        len = ldp(((size_t)cy << P.sx) + ic.cx1 + 1) - st;
      }
    }
    int x = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(~0u, x, o);
      if (lane >= o) x += y;
    }
    if (sidx < nseg) {
      sh->seg_start[b][sidx] = st;
      sh->seg_off[b][sidx] = base + x - len;
    }
    base += __shfl_sync(~0u, x, 31);
  }
  if (lane == 0) {
    sh->seg_off[b][nseg] = base;
    sh->nseg[b] = nseg;
    sh->rows_left[b] = full ? 0 : nrows - nseg;
  }
}

// Dynamic schedule: the stager's lane 0 takes the next ticket (band items in
// order, then kItemEnd).
__device__ __forceinline__ void ticket_item(const BandParams& P, long long t, int& kind, long long& idx) {
  idx = t - P.npro;
  kind = idx < P.total_items ? kItemBand : kItemEnd;
}

// `taken` >= 0: a ticket this CTA already holds (its first band item).
__device__ __forceinline__ void stage_next(const BandParams& P, BandShared* sh, int b, long long taken) {
  const int lane = threadIdx.x & 31;
  ItemCfg& ic = sh->ic[b];
  if (lane == 0) {
    int kind;
    long long idx;
    ticket_item(P, taken >= 0 ? taken : (long long)atomicAdd(P.ticket, 1), kind, idx);
    ic.kind = kind;
    ic.item = idx;
    if (kind == kItemBand) item_setup(P, idx, ic);
    else ic.pl = (int)idx;
  }
  __syncwarp();
  if (ic.kind == kItemBand) {
    item_stage(P, ic.item, sh, b, -2);
  } else if (lane == 0) {
    sh->nseg[b] = 0;
    sh->seg_off[b][0] = 0;
    sh->rows_left[b] = 0;
  }
}

// One regenerated particle, both frames (what the splat needs).
struct PFrames {
  int ax1, ay1, ax2, ay2;
  float fx1, fy1, fx2, fy2;
  float amp1, amp2, sig, sx2, sy2, rho1, rho2;
  bool on1, on2;
};

// Regenerate particle gi of seeding cell cc from its ParticleA draw `a`:
// position, advection, appearance, and whether each frame can touch the tile
// [r0, r1) x [c0, c1) (full patch window). `between` runs after the four flow
// loads are issued and before their values are used (the caller draws the
// next particle's Philox there, hiding the L2 latency of the loads).
template <class Between>
__device__ __forceinline__ void band_gen(const BandParams& P, const RngKey& key, const PairHdr& hd,
                                         const float2* __restrict__ flow, int gi, int cc, const uint4 a,
                                         int h, int r0, int r1, int c0, int c1, PFrames& o,
                                         Between between) {
  const GenCfg& g = P.g;
  const int CX = 1 << P.sx;
  const uint32_t X = cell_coord((uint32_t)(cc & (CX - 1)), a.x, g.W, P.sx);
  const uint32_t Y = cell_coord((uint32_t)(cc >> P.sx), a.y, g.H, P.sy);
  fixed_anchor(X, o.ax1, o.fx1);
  fixed_anchor(Y, o.ay1, o.fy1);
  // advect (particles.py:129-136): bilinear, edge-clamped (flowfield.py:207-232)
  int fcx, fcy;
  float tx, ty;
  fixed_cell(X, g.W, fcx, tx);
  fixed_cell(Y, g.H, fcy, ty);
  // fcx <= W - 2 and fcy <= H - 2 (H, W >= 2): the four nodes are
  // fp[0], fp[1], fp[W], fp[W + 1]
  const float2* fp = flow + (fcy * g.W + fcx);
  const float2* fq = fp + g.W;
  const float2 q00 = __ldg(fp), q01 = __ldg(fp + 1);
  const float2 q10 = __ldg(fq), q11 = __ldg(fq + 1);
  const float d = lerpf_exact(g.d_lo, g.d_span, q_to_unit(diam_q(hd, gi, a.z)));
  const float i0 = lerpf_exact(g.i0_lo, g.i0_span, unit23(a.w));
  o.sig = __fmul_rn(d, g.inv_ratio);
  Look lk;
  seed_look(g, key, gi, o.sig, i0, lk);
  o.amp1 = lk.amp1; o.amp2 = lk.amp2;
  o.sx2 = lk.sx2; o.sy2 = lk.sy2;
  o.rho1 = lk.rho1; o.rho2 = lk.rho2;
  // anchor rows [r0 - h, r1 + h) and columns [c0 - h, c1 + h) reach the tile
  const bool in1 = (unsigned)(o.ay1 - (r0 - h)) < (unsigned)(r1 - r0 + 2 * h) &&
                   (unsigned)(o.ax1 - (c0 - h)) < (unsigned)(c1 - c0 + 2 * h);
  o.on1 = in1 && lk.vis1 && lk.amp1 > 0.f;
  between(o);   // frame-1 work while the flow loads are in flight
  const float u = bilerp(q00.x, q01.x, q10.x, q11.x, tx, ty);
  const float v = bilerp(q00.y, q01.y, q10.y, q11.y, tx, ty);
  advect_anchor(X, o.ax1, u, o.ax2, o.fx2);
  advect_anchor(Y, o.ay1, v, o.ay2, o.fy2);
  const bool in2 = (unsigned)(o.ay2 - (r0 - h)) < (unsigned)(r1 - r0 + 2 * h) &&
                   (unsigned)(o.ax2 - (c0 - h)) < (unsigned)(c1 - c0 + 2 * h);
  o.on2 = in2 && lk.vis2 && lk.amp2 > 0.f;
}

__device__ __forceinline__ uint4 draw_a(const GenCfg& g, const RngKey& key, int gi) {
  return philox_rk(make_uint4((uint32_t)gi, key.pair, key.batch, kTagParticleA), g.rk);
}

// Worker warps: regenerate, advect and splat the particles of one item
// (variant fixed per item, see ItemCfg::var). NTW worker threads; BAR is the
// workers' own named barrier (rare multi-pass staging).
template <int PSF, int SEP, int WM, int NTW = kBandThreads, int BAR = 1>
__device__ __forceinline__ void band_particles(const BandParams& P, BandShared* sh, int buf, long long item,
                                               int* acc0, int* acc1) {
  const int tid = threadIdx.x, warp = tid >> 5;
  const ItemCfg& ic = sh->ic[buf];
  const int pl = ic.pl;
  const int r0 = ic.r0, r1 = ic.r1, c0 = ic.c0, c1 = ic.c1;
  const int h = ic.h, shift = ic.shift;
  const PairHdr& hd = ic.hd;
  const float scale = (float)(1 << shift);
  const float2* flow = P.flows + (size_t)ic.field * P.field_elems;
  const unsigned short* cof = P.cell_of + (size_t)pl * cof_stride(P.n);
  const RngKey key = band_key(P, pl);
  int next_row = ic.cy0;   // first cell row of the current pass
  for (;;) {
    const int nseg = sh->nseg[buf];
    const int N = sh->seg_off[buf][nseg];
    const int* soff = sh->seg_off[buf];
    const int* sst = sh->seg_start[buf];
    // slot q (clamped into [0, N)) -> particle index (segment search)
    const int sst0 = sst[0];
    auto locate = [&](int q) {
      q = min(q, N - 1);
      if (nseg == 1) return sst0 + q;
      int sg = 0;
      {
        int hi = nseg - 1;
        while (sg < hi) {
          const int mid = (sg + hi + 1) >> 1;
          if (soff[mid] <= q) sg = mid;
          else hi = mid - 1;
        }
      }
      return sst[sg] + (q - soff[sg]);
    };
    {
      // software pipeline: the Philox draw of the next slot is computed while
      // this slot's flow loads are in flight; its cell load one slot ahead
      int gA = 0, cA = 0;
      uint4 aA = make_uint4(0, 0, 0, 0);
      if (N > 0) {
        gA = locate(tid);
        cA = __ldcg(cof + gA);
        aA = draw_a(P.g, key, gA);
      }
      for (int qb = 0; qb < N; qb += NTW) {
        const int qa = qb + tid;
        const int giA = gA, ccA = cA;
        const uint4 a = aA;
        const bool more = qb + NTW < N;
        if (more) {
          gA = locate(qa + NTW);
          cA = __ldcg(cof + gA);
        }
        PFrames A;
        const bool ok = qa < N;
        band_gen(P, key, hd, flow, giA, ccA, a, h, r0, r1, c0, c1, A, [&](const PFrames& F) {
          if (ok && F.on1)
            splat_v<PSF, SEP, WM>(acc0, P.AS, F.ax1, F.ay1, F.fx1, F.fy1, F.amp1, F.sig, F.sig, F.rho1, h, r0,
                                  r1, c0, c1, shift, scale);
          if (more) aA = draw_a(P.g, key, gA);
        });
        if (ok) {
          if (A.on2)
            splat_v<PSF, SEP, WM>(acc1, P.AS, A.ax2, A.ay2, A.fx2, A.fy2, A.amp2, A.sx2, A.sy2, A.rho2, h, r0,
                                  r1, c0, c1, shift, scale);
        }
        __syncwarp();
      }
    }
    if (sh->rows_left[buf] <= 0) break;
    // rare: more cell rows than one segment table -> worker warp 0 stages
    // the next rows of this item (named barrier: workers only)
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NTW));
    next_row += kMaxSeg;
    if (warp == 0) item_stage(P, item, sh, buf, next_row);
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NTW));
  }
}


// ----------------------------------------------------------------------------
// Bank-sorted splat for large windows (C3: d up to 4 px, 12 x 12 windows).
// With one particle-frame per lane, the 32 lanes of a shared-memory atomic hit
// random banks (measured 3.7 wavefronts per ATOMS at C3: the shared-atomic
// pipe, not the SFU, bounded the kernel). Here the workers first turn their
// particle-frames into splat records (window origin, extents, Gaussian
// coefficients), counting-sort them by (window class, accumulator bank of the
// window origin), then splat in rounds where lane l takes record r + l*R of
// the class (R = ceil(n / 32)): lanes of one round sit in different banks,
// and every slot (i, j) of the round shifts all lanes by the same i*AS + j,
// so each ATOMS is (nearly) conflict-free. The class bounds the unpredicated
// window (4, 6, 8, 10, 12) instead of the pair's maximum. Same per-slot values
// as splat_sep_u.
// ----------------------------------------------------------------------------

struct __align__(16) SplatRec {
  int base;        // accumulator offset of the window origin (frame 2: + TH * AS)
  int nrnc;        // rows | cols << 16 inside the tile
  float dx0, dy0, A, C, Ls, pad;
};

constexpr int kSortPPT = 2;        // particles per worker thread per sorted chunk

struct __align__(16) SortShared {
  SplatRec rec[2 * kSortPPT * kBandThreads];          // record of (thread, particle, frame), unsorted
  unsigned short idx[2 * kSortPPT * kBandThreads];    // sorted order -> record
  int cnt[kSortClasses * 32];                // (class, bank) counts
  int cls_start[kSortClasses + 1];           // class starts in sorted order
  int cls_round[kSortClasses + 1];           // prefix of rounds per class
};

// Record of one separable particle-frame; returns its sort key or -1 (no pixel
// of the tile in the window). The class bounds the unpredicated WM x WM
// window; a window that would run past the frame's TH accumulator rows starts
// higher instead (its rows above the particle's window get Y = 0), so the
// sorted path needs no padding rows behind the accumulators.
__device__ __forceinline__ int make_rec(int f_off, int AS, int TH, int ax, int ay, float fx, float fy,
                                        float amp, float sx, float sy, int h, int r0, int r1, int c0, int c1,
                                        int shift, SplatRec& r) {
  const float R = __fmul_rn(fmaxf(sx, sy), kTightR);
  int rlo, clo, nr, nc;
  if (!tile_window(ax, ay, fx, fy, R, h, r0, r1, c0, c1, rlo, clo, nr, nc)) return -1;
  const int w = max(nr, nc);
  const int cls = w <= 4 ? 0 : min(kSortClasses - 1, (w - 3) >> 1);   // 5-6: 1, 7-8: 2, 9-10: 3, 11-12: 4
  const int top = r0 + TH - (4 + 2 * cls);   // last origin row whose window stays in the frame
  const int off = (rlo > top && top >= r0) ? rlo - top : 0;
  rlo -= off;
  r.base = f_off + (rlo - r0) * AS + (clo - c0);
  r.nrnc = off | ((off + nr) << 8) | (nc << 16);
  r.dx0 = (float)(clo - ax) - fx;
  r.dy0 = (float)(rlo - ay) - fy;
  const float isx = rcp_approx(sx), isy = rcp_approx(sy);
  r.A = (0.5f * kLog2e) * isx * isx;
  r.C = (0.5f * kLog2e) * isy * isy;
  r.Ls = lg2_approx(amp) + (float)shift;
  r.pad = 0.f;
  return cls * 32 + (r.base & 31);
}

// One record, unpredicated WM x WM window (slots outside the record's window
// add exactly 0; rows [rlo, rhi) of the window carry the particle, columns
// past the tile's last row spill into the accumulator's slack words).
template <int WM>
__device__ __forceinline__ void splat_rec(int* __restrict__ acc, int AS, const SplatRec& r) {
  const int rlo = r.nrnc & 0xff, rhi = (r.nrnc >> 8) & 0xff, nc = r.nrnc >> 16;
  int* base = acc + r.base;
  float X[WM];
#pragma unroll
  for (int j = 0; j < WM; ++j) {
    const float dx = r.dx0 + (float)j;
    const float xv = ex2_approx(fmaf(-r.A * dx, dx, r.Ls));
    X[j] = j < nc ? xv : 0.f;
  }
  if constexpr (WM <= 8) {
    float Y[WM];
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      const float dy = r.dy0 + (float)i;
      const float yv = ex2_approx(-r.C * dy * dy);
      Y[i] = (i >= rlo && i < rhi) ? yv : 0.f;
    }
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      int* row = base + i * AS;
#pragma unroll
      for (int j = 0; j < WM; ++j)
        atomicAdd(row + j, __float_as_int(fmaf(X[j], Y[i], 12582912.0f)) - 0x4B400000);
    }
  } else {
#pragma unroll 1
    for (int i = 0; i < WM; ++i) {
      const float dy = r.dy0 + (float)i;
      const float yv = ex2_approx(-r.C * dy * dy);
      const float Y = (i >= rlo && i < rhi) ? yv : 0.f;
      int* row = base + i * AS;
#pragma unroll
      for (int j = 0; j < WM; ++j)
        atomicAdd(row + j, __float_as_int(fmaf(X[j], Y, 12582912.0f)) - 0x4B400000);
    }
  }
}

// Worker warps, sorted splat: per chunk (kSortPPT particles per worker
// thread), (1) regenerate and write records + count keys, (2) every warp
// scans the counts and scatters its records' sorted positions, (3) splat
// rounds, smallest class first (warp w takes rounds w, w + 8, ...). Three
// named barriers (BAR) per chunk. (Measured against a double-buffered variant
// that overlaps the generation of chunk k with the splat of chunk k-1: that
// one needs twice the record space, i.e. shorter tiles, and was slower.)
template <int PSF, int NTW = kBandThreads, int BAR = 1>
__device__ __forceinline__ void band_particles_sorted(const BandParams& P, BandShared* sh, SortShared* ss,
                                                      int buf, long long item, int* acc0) {
  constexpr int NWW = NTW / 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const ItemCfg& ic = sh->ic[buf];
  const int pl = ic.pl;
  const int r0 = ic.r0, r1 = ic.r1, c0 = ic.c0, c1 = ic.c1;
  const int h = ic.h, shift = ic.shift;
  const PairHdr& hd = ic.hd;
  const int AS = P.AS, f2off = P.TH * P.AS;
  const float2* flow = P.flows + (size_t)ic.field * P.field_elems;
  const unsigned short* cof = P.cell_of + (size_t)pl * cof_stride(P.n);
  const RngKey key = band_key(P, pl);
  int next_row = ic.cy0;
  for (;;) {
    const int nseg = sh->nseg[buf];
    const int N = sh->seg_off[buf][nseg];
    const int* soff = sh->seg_off[buf];
    const int* sst = sh->seg_start[buf];
    const int sst0 = sst[0];
    auto locate = [&](int q) {
      q = min(q, N - 1);
      if (nseg == 1) return sst0 + q;
      int sg = 0;
      {
        int hi = nseg - 1;
        while (sg < hi) {
          const int mid = (sg + hi + 1) >> 1;
          if (soff[mid] <= q) sg = mid;
          else hi = mid - 1;
        }
      }
      return sst[sg] + (q - soff[sg]);
    };
    int gA = 0, cA = 0;
    uint4 aA = make_uint4(0, 0, 0, 0);
    if (N > 0) {
      gA = locate(tid);
      cA = __ldcg(cof + gA);
      aA = draw_a(P.g, key, gA);
    }
    for (int qc = 0; qc < N; qc += kSortPPT * NTW) {
      int kk[2 * kSortPPT], rk[2 * kSortPPT];
#pragma unroll
      for (int p = 0; p < kSortPPT; ++p) {
        const int qb = qc + p * NTW;
        const int qa = qb + tid;
        const int giA = gA, ccA = cA;
        const uint4 a = aA;
        const bool more = qb + NTW < N;
        if (more) {
          gA = locate(qa + NTW);
          cA = __ldcg(cof + gA);
        }
        PFrames A;
        const bool ok = qa < N;
        int k1 = -1, k2 = -1, rk1 = 0, rk2 = 0;
        const int slot = 2 * (p * NTW + tid);
        band_gen(P, key, hd, flow, giA, ccA, a, h, r0, r1, c0, c1, A, [&](const PFrames& F) {
          if (ok && F.on1) {
            SplatRec r;
            k1 = make_rec(0, AS, P.TH, F.ax1, F.ay1, F.fx1, F.fy1, F.amp1, F.sig, F.sig, h, r0, r1, c0, c1, shift, r);
            if (k1 >= 0) {
              ss->rec[slot] = r;
              rk1 = atomicAdd(&ss->cnt[k1], 1);
            }
          }
          if (more) aA = draw_a(P.g, key, gA);
        });
        if (ok && A.on2) {
          SplatRec r;
          k2 = make_rec(f2off, AS, P.TH, A.ax2, A.ay2, A.fx2, A.fy2, A.amp2, A.sx2, A.sy2, h, r0, r1, c0, c1, shift, r);
          if (k2 >= 0) {
            ss->rec[slot + 1] = r;
            rk2 = atomicAdd(&ss->cnt[k2], 1);
          }
        }
        kk[2 * p] = k1; rk[2 * p] = rk1;
        kk[2 * p + 1] = k2; rk[2 * p + 1] = rk2;
      }
      asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NTW) : "memory");   // counts final
      {
        // (class, bank) starts: every warp scans the counts itself (no serial
        // step), then scatters its own records' sorted positions
        int st[kSortClasses], tots[kSortClasses];
        int base = 0;
#pragma unroll
        for (int c = 0; c < kSortClasses; ++c) {
          const int v = ss->cnt[c * 32 + lane];
          int x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(~0u, x, o);
            if (lane >= o) x += y;
          }
          st[c] = base + x - v;
          tots[c] = __shfl_sync(~0u, x, 31);
          base += tots[c];
        }
#pragma unroll
        for (int e = 0; e < 2 * kSortPPT; ++e) {
          int sv = 0;
#pragma unroll
          for (int c = 0; c < kSortClasses; ++c) {
            const int a1 = __shfl_sync(~0u, st[c], kk[e] & 31);
            if ((kk[e] >> 5) == c) sv = a1;
          }
          if (kk[e] >= 0) ss->idx[sv + rk[e]] = (unsigned short)(2 * ((e >> 1) * NTW + tid) + (e & 1));
        }
        if (tid == 0) {
          int b0 = 0, rounds = 0;
#pragma unroll
          for (int c = 0; c < kSortClasses; ++c) {
            ss->cls_start[c] = b0;
            ss->cls_round[c] = rounds;
            b0 += tots[c];
            rounds += (tots[c] + 31) >> 5;
          }
          ss->cls_start[kSortClasses] = b0;
          ss->cls_round[kSortClasses] = rounds;
        }
      }
      asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NTW) : "memory");   // sorted order published
      for (int e = tid; e < kSortClasses * 32; e += NTW) ss->cnt[e] = 0;   // every warp has read them
      // class layout in registers (the round -> class search is per round)
      int cr[kSortClasses + 1];
#pragma unroll
      for (int c = 0; c <= kSortClasses; ++c) cr[c] = ss->cls_round[c];
      const int nrounds = cr[kSortClasses];
      for (int rr = warp; rr < nrounds; rr += NWW) {
        int c = 0;
#pragma unroll
        for (int t = 1; t < kSortClasses; ++t) c += rr >= cr[t];
        int c0 = cr[0], c1 = cr[1];
#pragma unroll
        for (int t = 1; t < kSortClasses; ++t)
          if (c == t) { c0 = cr[t]; c1 = cr[t + 1]; }
        const int R = c1 - c0;
        const int cs = ss->cls_start[c];
        const int k = (rr - c0) + lane * R;
        if (k < ss->cls_start[c + 1] - cs) {
          const SplatRec r = ss->rec[ss->idx[cs + k]];
          switch (c) {   // warp-uniform
            case 0: splat_rec<4>(acc0, AS, r); break;
            case 1: splat_rec<6>(acc0, AS, r); break;
            case 2: splat_rec<8>(acc0, AS, r); break;
            case 3: splat_rec<10>(acc0, AS, r); break;
            default: splat_rec<12>(acc0, AS, r); break;
          }
        }
      }
      asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NTW) : "memory");
    }
    if (sh->rows_left[buf] <= 0) break;
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NTW) : "memory");
    next_row += kMaxSeg;
    if (warp == 0) item_stage(P, item, sh, buf, next_row);
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NTW) : "memory");
  }
}

// Workers: particles of the staged item `buf`, then the fused epilogue; two
// block barriers (the staging warp meets them).
template <int PSF, int SORT>
__device__ __forceinline__ void render_item(const BandParams& P, BandShared* sh, SortShared* ss, int buf,
                                            int* acc0, int* acc1) {
  const ItemCfg& ic = sh->ic[buf];
  const long long item = ic.item;
  if (threadIdx.x >= kBandThreads) {
    // staging warp: the next item, then the store of this one (below)
    stage_next(P, sh, buf ^ 1, -1);
  } else if constexpr (PSF == kPsfErf) {
    band_particles<PSF, 0, 0>(P, sh, buf, item, acc0, acc1);
  } else {
    switch (ic.var) {
      case kVarSorted:
        if constexpr (SORT != 0) band_particles_sorted<PSF>(P, sh, ss, buf, item, acc0);
        break;
#define PGB_V(S, W) case 16 * S + W: band_particles<PSF, S, W>(P, sh, buf, item, acc0, acc1); break;
      PGB_V(1, 1) PGB_V(1, 2) PGB_V(1, 3) PGB_V(1, 4) PGB_V(1, 5) PGB_V(1, 6)
#undef PGB_V
      default: band_particles<PSF, 0, 0>(P, sh, buf, item, acc0, acc1); break;
    }
  }
#ifdef PGB_TRACE
  trace_item(0);
#endif
  __syncthreads();   // particles done (stager: next item staged)
#ifdef PGB_TRACE
  trace_item(1);
#endif
  const int pl = ic.pl;
  const int r0 = ic.r0, r1 = ic.r1, c0 = ic.c0, c1 = ic.c1;
  const float inv_scale = 1.0f / (float)(1 << ic.shift);
  band_store(P, acc0, pl, 0, r0, r1 - r0, c0, c1 - c0, inv_scale);
  band_store(P, acc1, pl, 1, r0, r1 - r0, c0, c1 - c0, inv_scale);
  __syncthreads();   // accumulators zeroed
#ifdef PGB_TRACE
  trace_item(2);
  if (threadIdx.x == 0) ++g_trace_item;
#endif
}

// SORT = 1: the body for plans with a record region (large windows), in a
// separate kernel so the sorted splat's registers do not weigh on the
// small-window particle loop.
template <int PSF, int SORT>
__device__ __forceinline__ void band_body(const BandParams& P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BandShared* sh = reinterpret_cast<BandShared*>(smem_raw);
  SortShared* ss = reinterpret_cast<SortShared*>(smem_raw + sizeof(BandShared));   // when rec_bytes > 0
  int* acc0 = reinterpret_cast<int*>(smem_raw + sizeof(BandShared) + P.rec_bytes);
  int* acc1 = acc0 + P.TH * P.AS;
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool stager = warp == kBandWarps;   // the extra warp stages items, workers splat + store
  // the prologue borrows the record + accumulator region (>= its histogram, see make_band_plan)
  const int acc_bytes = P.pro_smem;
  int* bins = reinterpret_cast<int*>(ss);
  auto zero_acc = [&]() {
    // (workers) both frame accumulators + the zero padding behind them (the
    // prologue borrowed them), sorted-splat counts
    for (int e = tid; e < ((2 * P.TH + P.pad_rows) * P.AS + 16) / 4; e += kBandThreads)
      reinterpret_cast<int4*>(acc0)[e] = make_int4(0, 0, 0, 0);
    if (P.rec_bytes)
      for (int e = tid; e < kSortClasses * 32; e += kBandThreads) ss->cnt[e] = 0;
  };
  PGB_STAMP(0);
#ifdef PGB_TRACE
  if (tid == 0) {
    g_trace_first = 0, g_trace_item = 0;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (blockIdx.x < 2048) g_trace[blockIdx.x * kTraceSlots + 39] = smid + 1;
  }
#endif
  if (blockIdx.x == gridDim.x - 1 && P.zero_head)
    for (int e = tid; e < P.zero_head_n; e += kBandBlock) P.zero_head[e] = make_int4(0, 0, 0, 0);
  // One ticket sequence: [0, npro) prologue items (the flow-bound chunks,
  // histogram parts, pair prologues, particle -> cell windows), then the band
  // items. Every ticket waits only on earlier tickets (a prologue on its
  // histogram parts, a window on its pair's prefix, band items on pair and
  // field flags), each taken by a running CTA: forward progress without
  // co-residency (MPS limits, green contexts, a concurrent kernel holding SMs,
  // any grid size).
  const int nfc = P.field_cnt * kFieldBlocks;
  long long first;
  if (tid == 0) sh->ticket0 = atomicAdd(P.ticket, 1);
  if (tid == kBandThreads) touch_stage_params(P);
  __syncthreads();
  first = sh->ticket0;
  for (;;) {
    if (first >= P.npro) break;
    // take the following ticket now (its atomic round trip overlaps this item;
    // it is later than `first`, and every item waits only on earlier tickets,
    // so the smallest unfinished ticket is always some CTA's current item)
    if (tid == 0) sh->ticket_next = atomicAdd(P.ticket, 1);
    int w = (int)first;
    const int nparts = P.pro_parts > 1 ? P.pairs * P.pro_parts : 0;
    if (w < nfc) {
      field_bound_chunk<kBandBlock>(P, P.field_lo + w / kFieldBlocks, w % kFieldBlocks);
      PGB_STAMP(1);
    } else if ((w -= nfc) < nparts) {
      pair_hist_part<kBandBlock>(P, w / P.pro_parts, w % P.pro_parts, bins);
    } else if ((w -= nparts) < P.pairs) {
      pair_prologue<kBandBlock>(P, w, bins, acc_bytes);
    } else {
      w -= P.pairs;
      pair_fill_window<kBandBlock>(P, w / P.fill_wins, w % P.fill_wins, bins);
    }
    __syncthreads();
    first = sh->ticket_next;
    __syncthreads();
  }
  // dynamic schedule: the staging warp takes the ticket of item k+1 and
  // prepares it (parameters + particle segments) while the workers splat item
  // k; the first item is staged while the workers zero the accumulators
  PGB_STAMP(8);
  if (stager) stage_next(P, sh, 0, first);
  else zero_acc();
  __syncthreads();
  PGB_STAMP(9);
#ifdef PGB_TRACE
  int nitems = 0;
#endif
  for (int buf = 0;; buf ^= 1) {
    const int kind = sh->ic[buf].kind;
    if (kind == kItemEnd) break;
#ifdef PGB_TRACE
    ++nitems;
#endif
    render_item<PSF, SORT>(P, sh, ss, buf, acc0, acc1);
  }
  PGB_STAMP(12);
#ifdef PGB_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 2048) g_trace[blockIdx.x * kTraceSlots + 13] = nitems;
#endif
}


template <int PSF>
__global__ void PGB_BAND_BOUNDS band_kernel(const BandParams P) {
  band_body<PSF, 0>(P);
}

// Large windows (a separate kernel: its chunk state costs registers, 96 with
// a few spills at 2 CTAs x 9 warps per SM -- five warps of one SM sub-
// partition share 16 K registers, so 104 would drop it to one CTA per SM).
__global__ void PGB_BAND_BOUNDS band_sorted_kernel(const BandParams P) {
  band_body<kPsfPoint, 1>(P);
}

// Particle arrays of the generator (one block per pair): exactly the particles
// the band kernel renders (positions = anchor + fraction).
__global__ void sample_band_kernel(const BandParams P, pgb_particle_out O) {
  const int pl = blockIdx.x;
  PGB_STAMP(9);
  const PairHdr hd = P.hdr[pl];
  const int ncell = 1 << (P.sy + P.sx);
  const int* pre = P.prefix + (size_t)pl * pre_stride(ncell);
  const float2* flow = P.flows + (size_t)((P.pair_base + pl) / P.pairs_per_field) * P.field_elems;
  for (int gi = threadIdx.x; gi < P.n; gi += blockDim.x) {
    int cy = 0, cx = 0;
    if (gi < hd.M) {
      int lo = 0, hi = ncell - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(pre + mid) <= gi) lo = mid;
        else hi = mid - 1;
      }
      cy = lo >> P.sx;
      cx = lo & ((1 << P.sx) - 1);
    }
    Particle pt;
    seed_particle(P, hd, pl, gi, cy, cx, flow, pt);
    const size_t o = (size_t)pl * P.n + gi;
    const Frame& a = pt.fr[0];
    const Frame& b = pt.fr[1];
    if (O.pos1) { O.pos1[2 * o] = (double)a.ax + (double)a.fx; O.pos1[2 * o + 1] = (double)a.ay + (double)a.fy; }
    if (O.pos2) { O.pos2[2 * o] = (double)b.ax + (double)b.fx; O.pos2[2 * o + 1] = (double)b.ay + (double)b.fy; }
    if (O.i0_1) O.i0_1[o] = a.amp;
    if (O.sx_1) O.sx_1[o] = a.sx;
    if (O.sy_1) O.sy_1[o] = a.sy;
    if (O.rho_1) O.rho_1[o] = a.rho;
    if (O.i0_2) O.i0_2[o] = b.amp;
    if (O.sx_2) O.sx_2[o] = b.sx;
    if (O.sy_2) O.sy_2[o] = b.sy;
    if (O.rho_2) O.rho_2[o] = b.rho;
    if (O.diameter) O.diameter[o] = pt.diam;
    if (O.z1) O.z1[o] = pt.z1;
    if (O.active) O.active[o] = pt.active ? 1 : 0;
    if (O.visible1) O.visible1[o] = pt.vis1 ? 1 : 0;
    if (O.visible2) O.visible2[o] = pt.vis2 ? 1 : 0;
  }
  PGB_STAMP(10);
}

}  // namespace pgb
