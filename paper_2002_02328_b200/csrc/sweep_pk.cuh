// Persistent block-Jacobi sweep: the whole bd3mg_jacobi_sweep (recorder,
// regulariser gradient, residual, gradient, Gram, solve, update) as ONE
// launch of one CTA per resident slot (148 SMs x 3), pulling work items from
// a queue in a precomputed topological order and waiting on per-plane /
// per-block completion counters instead of kernel boundaries.
//
// Why: in the multi-kernel sweep each correlation phase ends in a partial
// last wave (1024 tiles on 444 slots), the phases are serialised by their
// dependencies, and the HBM-bound stencils cannot share SMs with the
// correlations (shared memory is full).  Here a GRAD tile of block 0 starts
// as soon as the residual planes it reads are done -- while the residual of
// the far planes is still running -- and a slot that would idle in a tail
// takes the next ready item of any phase: stencil items run next to
// correlation tiles on the same SM.
//
// Items (one CTA each, 128 threads):
//   GREG (b, tile)        greg_tile: omega, regulariser gradient, recorder terms, snapshot roll
//   RESID (plane, tile)   conv_tile M_RESID: r = H x - y, sum r^2
//   GRAD (b, plane, tile) conv_tile M_GRAD (adjoint): g = H^T r + greg
//   RG (b, chunk, tile)   reg_gram_tile: regulariser Gram terms, rhs, flags
//   GRAM (b, plane, tile) conv_tile M_GRAM2P: <Hg,Hg>, <Hg,Hd>, <Hd,Hd> (two passes over one tile ring)
//   SOLVE (b)             final Gram / rhs reductions + the 2x2 solve (solve_one)
//   UPD (b, chunk)        x += inc, d = inc (+ mirror stores into peer halo inboxes)
//   RED (0|1)             recorder sums (stencil terms | data term); the later one writes the terms
// Every item runs the same device function as the multi-kernel path with
// the same tile -> partial-row mapping, and every final reduction replays
// the 256-thread tree of reduce_rows / reduce_solve, so the sweep is bitwise
// that of bd3mg_jacobi_sweep's multi-kernel path (tests/test_gpu_sweep_pk.py).
//
// Deadlock freedom: items are dequeued in one global order (atomic ticket)
// and every dependency of an item lies earlier in that order, so an item a
// CTA waits on has already been taken by a running CTA whose own
// dependencies are earlier still.
//
// Memory ordering: producers write with generic stores, then every thread
// fences (gpu scope + async proxy) before the CTA bumps the completion
// counter with a release; consumers acquire the counter, then fence the
// async proxy before their TMA loads; produced data read with generic loads
// goes through L2 (ld.cg) -- L1 is not coherent across SMs.
#pragma once

#include <cuda.h>

#include "depthvar.cuh"
#include "solver.cuh"
#include "stencil_tma.cuh"

namespace bd3mg {

enum PkType : int { PK_GREG = 0, PK_RESID = 1, PK_GRAD = 2, PK_RG = 3, PK_GRAM = 4, PK_SOLVE = 5, PK_UPD = 6, PK_RED = 7 };

struct PkSeg {
  uint32_t first;  // queue index of the segment's first item
  uint16_t z;      // plane (RESID/GRAD/GRAM), first tile (GREG/RG), first chunk (UPD), which (RED)
  uint16_t aux;    // RESID/GRAD/GRAM: first tile; RG: chunk index
  uint8_t type, b;
};

constexpr int kPkMaxSeg = 1700;
// rows per thread of the residual / gradient tiles: 8 (64 x 32 tiles, like
// the Gram) halves the staging ring, so 4 CTAs share an SM -- three keep the
// FMA pipe fed while the fourth runs a memory-bound item
#ifndef BD3MG_PK_RY
#define BD3MG_PK_RY 8
#endif
constexpr int kPkRY = BD3MG_PK_RY;
// 4 slots cap the registers at 128 and the kernel then spills; measured on
// B200: spilled values were corrupted across items (tests/test_gpu_sweep_pk.py
// fails at 4, passes at 3), so 3 is the default
#ifndef BD3MG_PK_SLOTS
#define BD3MG_PK_SLOTS 3
#endif
template <typename T, int K>
constexpr int pk_slots_per_sm() { return (sizeof(T) == 8 && K >= 9) ? 2 : (K >= 7 ? 3 : BD3MG_PK_SLOTS); }

// counter layout (ints): [0] ticket, [1] RED arrivals, then per block
// greg / grad / rg / gram / solve, then per residual plane
constexpr int kPkCtrTicket = 0, kPkCtrRed = 1, kPkCtrBlk = 2;
BD3MG_HD int pk_ctr_greg(int b) { return kPkCtrBlk + 5 * b + 0; }
BD3MG_HD int pk_ctr_grad(int b) { return kPkCtrBlk + 5 * b + 1; }
BD3MG_HD int pk_ctr_rg(int b) { return kPkCtrBlk + 5 * b + 2; }
BD3MG_HD int pk_ctr_gram(int b) { return kPkCtrBlk + 5 * b + 3; }
BD3MG_HD int pk_ctr_solve(int b) { return kPkCtrBlk + 5 * b + 4; }
BD3MG_HD int pk_ctr_resid(int zrel) { return kPkCtrBlk + 5 * kMaxJobs + zrel; }
BD3MG_HD int pk_ctr_count(int nres) { return kPkCtrBlk + 5 * kMaxJobs + nres; }

template <typename T>
struct PkArgs {
  ConvGeom<T> cg;
  StGeom<T> sg;
  // TMA maps (one per tensor and box shape)
  CUtensorMap tm_x;     // x fragment (plane 0 = frag_z0), correlation box   RESID input
  CUtensorMap tm_y;     // y rows (plane 0 = u_lo), TX x TY box               RESID epilogue
  CUtensorMap tm_r;     // r rows (plane 0 = u_lo), correlation box           GRAD input
  CUtensorMap tm_greg;  // greg rows (plane 0 = rec_lo), TX x TY box          GRAD epilogue
  CUtensorMap tm_g;     // g rows (plane 0 = rec_lo), Gram box                GRAM pass 1
  CUtensorMap tm_d;     // d fragment (plane 0 = frag_z0), Gram box           GRAM pass 0
  CUtensorMap tm_xs;    // x fragment, GregGeo box                            GREG
  CUtensorMap tm_gs;    // g rows, RgGeo box                                  RG
  CUtensorMap tm_ds;    // d fragment, RgGeo box                              RG
  const T* x;           // fragment (plane 0 = frag_z0), updated in place
  T* xw;
  long long frag_z0;
  int nzf;
  const T* y;           // y + z*plane = observation row z
  T* r;                 // residual rows [u_lo, u_hi]
  int u_lo, u_hi;
  T* g;                 // block rows [rec_lo, rec_hi] (all blocks back to back)
  T* greg;
  T* omega;
  int rec_lo, rec_hi;
  T* dmem;              // fragment-aligned memory store, updated in place
  T* snap;              // recorder rows, rolled by GREG
  double* eparts;       // GREG partial rows: (b * st_ty + by) * st_tx + bx
  double* cparts;       // RESID partial rows: (z - u_lo) * conv_tiles + t
  double* gparts;       // GRAM partial rows: g_row0[b] + (zo - olo_b) * gram_tiles + t
  double* rparts;       // RG partial rows: rg_row0[b] + (chunk * st_tiles + t)
  double* sums;         // [0] data sum, [1..5] stencil sums
  double* terms;        // the recorder terms of the anchor
  double* info;         // StepInfo per block
  int* ctr;
  int nb;
  int lo[kMaxJobs], hi[kMaxJobs], olo[kMaxJobs];
  int rg_c[kMaxJobs];   // z-chunk of the block's regulariser-Gram march
  long long g_row0[kMaxJobs], rg_row0[kMaxJobs];
  int conv_tx, conv_tiles, gram_tx, gram_tiles, st_tx, st_tiles;
  long long upd_chunk;  // elements per UPD item
  double fin_eta, fin_lam, fin_kappa;
  SolveArgs solve;      // (g_begin / r_begin ranges unused: rows from g_row0 / rg_row0)
  MirArgs<T, kMaxMirSegs> mir;
  int bar_off;          // PkCfg::data_bytes(kz): offset of the mbarriers / ticket in shared memory
  unsigned long long* trace;  // optional (BD3MG_PK_TRACE=1): per item [dequeued, deps met, done] ns + (sm, type, b, z)
  int nseg;
  uint32_t total;
  PkSeg seg[kPkMaxSeg];
};

// ---- synchronisation helpers ---------------------------------------------
BD3MG_D int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
BD3MG_D void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
BD3MG_D void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }
BD3MG_D void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
BD3MG_D void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// thread 0: wait until *p >= need
BD3MG_D void pk_wait(const int* p, int need) {
  if (need <= 0) return;
  int ns = 32;
  while (ld_acquire(p) < need) {
    __nanosleep(ns);
    ns = min(ns * 2, 256);
  }
}

// 256-thread deterministic row sum (reduce_rows_kernel / reduce_solve_kernel's
// cta_sum_rows) replayed by a 128-thread CTA: thread t plays threads t and
// t + 128 (same stride classes, same butterflies, same warp order).
BD3MG_D void pk_sum_rows(const double* __restrict__ rows, int nv, long long begin, long long end, double* s,
                         double* res) {
  double a0[kRedMaxNV], a1[kRedMaxNV];
#pragma unroll
  for (int k = 0; k < kRedMaxNV; ++k) { a0[k] = 0.0; a1[k] = 0.0; }
  for (long long r = begin + threadIdx.x; r < end; r += kEwNT) {
#pragma unroll
    for (int k = 0; k < kRedMaxNV; ++k)
      if (k < nv) a0[k] += __ldcg(rows + r * nv + k);
  }
  for (long long r = begin + threadIdx.x + kEwNT / 2; r < end; r += kEwNT) {
#pragma unroll
    for (int k = 0; k < kRedMaxNV; ++k)
      if (k < nv) a1[k] += __ldcg(rows + r * nv + k);
  }
#pragma unroll
  for (int k = 0; k < kRedMaxNV; ++k) {
    if (k < nv) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        a0[k] += __shfl_xor_sync(0xffffffffu, a0[k], off);
        a1[k] += __shfl_xor_sync(0xffffffffu, a1[k], off);
      }
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;  // virtual warps `warp` and `warp + 4`
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kRedMaxNV; ++k)
      if (k < nv) {
        s[k * 8 + warp] = a0[k];
        s[k * 8 + warp + 4] = a1[k];
      }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kRedMaxNV; ++k) {
    if (k < nv) {
      double t = s[k * 8];
#pragma unroll
      for (int w = 1; w < 8; ++w) t += s[k * 8 + w];
      res[k] = t;
    }
  }
  __syncthreads();
}

template <typename T>
BD3MG_D void pk_mirror_store(const MirArgs<T, kMaxMirSegs>& m, int blk, long long i, T v) {
  for (int j = 0; j < m.n; ++j) {
    const MirSeg<T>& s = m.s[j];
    if (s.blk == blk && i >= s.a && i < s.b) s.dst[i - s.a] = v;
  }
}

template <typename T, int K>
struct PkCfg {
  using CR = ConvCfg<T, K, K, M_RESID, kPkRY>;
  using CG = ConvCfg<T, K, K, M_GRAD, kPkRY>;
  using CM = ConvCfg<T, K, K, M_GRAM2P>;
  static constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
  // bytes any item uses from the aligned base (stencil layouts: their smem() minus its alignment slack;
  // the final reductions' scratch, 12 x 8 doubles, fits inside any of them)
  static size_t data_bytes(int kz) {
    const size_t st = cmax(GregGeo<T>::smem(), RgGeo<T>::smem()) - 128;
    return (cmax(cmax(CR::layout_bytes(kz), CG::layout_bytes(kz)), cmax(CM::layout_bytes(kz), st)) + 15) &
           ~size_t(15);
  }
  // [item data][4 mbarriers + ticket] after up to 128 bytes of alignment slack: 3 CTAs per SM at
  // 5x5 taps in fp64 (76 736 bytes)
  static size_t smem_bytes(int kz) { return 128 + data_bytes(kz) + 48; }
};

// 3 CTAs per SM where the staging ring allows it (fp64 3x3 / 5x5 taps), else 2
template <typename T, int K>
__global__ void __launch_bounds__(128, pk_slots_per_sm<T, K>())
    sweep_pk_kernel(const __grid_constant__ PkArgs<T> p) {
  using Cfg = PkCfg<T, K>;
  static_assert(sizeof(PkArgs<T>) <= 32000, "kernel parameter space");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* sbase = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + p.bar_off);
  int* s_item = reinterpret_cast<int*>(bars + 4);
  double* s_red = reinterpret_cast<double*>(sbase);  // SOLVE / RED scratch (no tile data then)
  const int rz = (p.cg.kz - 1) / 2;
  int* ctr = p.ctr;

  for (;;) {
    if (threadIdx.x == 0) s_item[0] = atomicAdd(ctr + kPkCtrTicket, 1);
    __syncthreads();
    const int item = s_item[0];
    if (item >= (int)p.total) return;
    // segment of the item (binary search over first indices)
    int lo = 0, hi = p.nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((int)p.seg[mid].first <= item) lo = mid;
      else hi = mid - 1;
    }
    const PkSeg sg = p.seg[lo];
    const int k = item - (int)sg.first;
    const int type = sg.type, b = sg.b;
    unsigned long long t_deq = 0;
    if (p.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_deq));

    // ---- dependencies (thread 0 waits; the CTA follows at the barrier) ----
    if (threadIdx.x == 0) {
      if (type == PK_GRAD) {
        const int zi = sg.z;
        for (int z = max(p.u_lo, zi - rz); z <= min(p.u_hi, zi + rz); ++z)
          pk_wait(ctr + pk_ctr_resid(z - p.u_lo), p.conv_tiles);
        pk_wait(ctr + pk_ctr_greg(b), p.st_tiles);
      } else if (type == PK_RG) {
        pk_wait(ctr + pk_ctr_grad(b), (p.hi[b] - p.lo[b] + 1) * p.conv_tiles);
        pk_wait(ctr + pk_ctr_greg(b), p.st_tiles);
      } else if (type == PK_GRAM) {
        pk_wait(ctr + pk_ctr_grad(b), (p.hi[b] - p.lo[b] + 1) * p.conv_tiles);
      } else if (type == PK_SOLVE) {
        const int olo = p.olo[b], ohi = min(p.cg.nz_global - 1, p.hi[b] + rz);
        pk_wait(ctr + pk_ctr_gram(b), (ohi - olo + 1) * p.gram_tiles);
        const int h = p.hi[b] - p.lo[b] + 1;
        pk_wait(ctr + pk_ctr_rg(b), (h + p.rg_c[b] - 1) / p.rg_c[b] * p.st_tiles);
      } else if (type == PK_UPD) {
        pk_wait(ctr + pk_ctr_solve(b), 1);
        // every reader of this block's x rows at the anchor is done
        for (int z = max(p.u_lo, p.lo[b] - rz); z <= min(p.u_hi, p.hi[b] + rz); ++z)
          pk_wait(ctr + pk_ctr_resid(z - p.u_lo), p.conv_tiles);
        for (int bb = max(0, b - 1); bb <= min(p.nb - 1, b + 1); ++bb) pk_wait(ctr + pk_ctr_greg(bb), p.st_tiles);
      } else if (type == PK_RED) {
        if (sg.z == 0) {
          for (int bb = 0; bb < p.nb; ++bb) pk_wait(ctr + pk_ctr_greg(bb), p.st_tiles);
        } else {
          for (int z = p.rec_lo; z <= p.rec_hi; ++z) pk_wait(ctr + pk_ctr_resid(z - p.u_lo), p.conv_tiles);
        }
      }
      fence_proxy_async_global();  // produced data is read by TMA below
      fence_proxy_async_smem();     // smem written by the previous item is refilled by TMA below
      if (p.trace) {
        unsigned long long t_go, sm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_go));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(*reinterpret_cast<unsigned*>(&sm)));
        sm &= 0xffffffffull;
        unsigned long long* tr = p.trace + 4ull * item;
        tr[0] = t_deq;
        tr[1] = t_go;
        tr[3] = (sm << 48) | ((unsigned long long)type << 40) | ((unsigned long long)b << 32) |
                ((unsigned long long)sg.z << 16) | (unsigned long long)sg.aux;
      }
    }
    __syncthreads();

    int nbars = 0;
    int* done = nullptr;
    // ---- the item ----------------------------------------------------------
    if (type == PK_RESID) {
      const int zo = sg.z, t = sg.aux + k;
      const int tx = t % p.conv_tx, ty = t / p.conv_tx;
      TileIO<T> io;
      io.in0 = {&p.tm_x, p.x, p.frag_z0, p.nzf, p.frag_z0};
      io.in1 = io.in0;
      io.dst = p.r + (long long)(zo - p.u_lo) * p.cg.plane;
      io.sub = p.y + (long long)zo * p.cg.plane;
      io.tm_epi = &p.tm_y;
      io.epi_z = zo - p.u_lo;
      io.use_tma = true;
      using C = typename Cfg::CR;
      conv_tile<T, K, K, M_RESID, false, kPkRY>(p.cg, io, zo, tx * C::TX, ty * C::TY,
                                         p.cparts + ((long long)(zo - p.u_lo) * p.conv_tiles + t), sbase, bars);
      nbars = 2;
      done = ctr + pk_ctr_resid(zo - p.u_lo);
    } else if (type == PK_GRAD) {
      const int zi = sg.z, t = sg.aux + k;
      const int tx = t % p.conv_tx, ty = t / p.conv_tx;
      TileIO<T> io;
      io.in0 = {&p.tm_r, p.r, (long long)p.u_lo, p.u_hi - p.u_lo + 1, (long long)p.u_lo};
      io.in1 = io.in0;
      io.dst = p.g + (long long)(zi - p.rec_lo) * p.cg.plane;
      io.sub = p.greg + (long long)(zi - p.rec_lo) * p.cg.plane;
      io.tm_epi = &p.tm_greg;
      io.epi_z = zi - p.rec_lo;
      io.use_tma = true;
      using C = typename Cfg::CG;
      conv_tile<T, K, K, M_GRAD, true, kPkRY>(p.cg, io, zi, tx * C::TX, ty * C::TY, nullptr, sbase, bars);
      nbars = 2;
      done = ctr + pk_ctr_grad(b);
    } else if (type == PK_GRAM) {
      const int zo = sg.z, t = sg.aux + k;
      const int tx = t % p.gram_tx, ty = t / p.gram_tx;
      const int hb = p.hi[b] - p.lo[b] + 1;
      TileIO<T> io;
      // input 0 = g rows of the block, input 1 = its memory direction (both embedded: zero outside the block)
      io.in0 = {&p.tm_g, p.g + (long long)(p.lo[b] - p.rec_lo) * p.cg.plane, (long long)p.lo[b], hb,
                (long long)p.rec_lo};
      io.in1 = {&p.tm_d, p.dmem + (long long)(p.lo[b] - p.frag_z0) * p.cg.plane, (long long)p.lo[b], hb,
                p.frag_z0};
      io.dst = nullptr;
      io.sub = nullptr;
      io.tm_epi = nullptr;
      io.epi_z = 0;
      io.use_tma = true;
      using C = typename Cfg::CM;
      conv_tile<T, K, K, M_GRAM2P, false>(
          p.cg, io, zo, tx * C::TX, ty * C::TY,
          p.gparts + 3 * (p.g_row0[b] + (long long)(zo - p.olo[b]) * p.gram_tiles + t), sbase, bars);
      nbars = 2;
      done = ctr + pk_ctr_gram(b);
    } else if (type == PK_GREG) {
      const int t = sg.z + k;
      StJob<T> J;
      J.a = p.x; J.a_z0 = p.frag_z0; J.lo = p.lo[b]; J.hi = p.hi[b];
      const long long o = (long long)(p.lo[b] - p.rec_lo) * p.cg.plane;
      J.b = p.snap ? p.snap + o : nullptr;
      J.snap_out = p.snap ? p.snap + o : nullptr;
      J.out0 = p.greg + o; J.out1 = p.omega + o;
      J.w = nullptr; J.work_begin = 0; J.chunk = 0; J.blo = J.bhi = 0; J.tz_off = J.tz_off_b = 0;
      greg_tile<T, true>(p.sg, J, &p.tm_xs, t % p.st_tx, t / p.st_tx,
                         p.eparts + ((long long)b * p.st_tiles + t) * kEvalNV, sbase, bars);
      nbars = GregGeo<T>::RING;
      done = ctr + pk_ctr_greg(b);
    } else if (type == PK_RG) {
      const int t = sg.z + k, chunk = sg.aux;
      const int c = p.rg_c[b];
      const int clo = p.lo[b] + chunk * c, chi = min(p.hi[b], clo + c - 1);
      const long long o = (long long)(clo - p.rec_lo) * p.cg.plane;
      StJob<T> J;
      J.a = p.g + o; J.a_z0 = clo;
      J.b = p.dmem + (long long)(clo - p.frag_z0) * p.cg.plane;
      J.w = p.omega + o;
      J.lo = clo; J.hi = chi;
      J.chunk = c < p.hi[b] - p.lo[b] + 1 ? 1 : 0;
      J.blo = p.lo[b]; J.bhi = p.hi[b];
      J.tz_off = clo - p.rec_lo; J.tz_off_b = clo - (int)p.frag_z0;
      J.out0 = J.out1 = nullptr; J.snap_out = nullptr; J.work_begin = 0;
      reg_gram_tile<T, true>(p.sg, J, &p.tm_gs, &p.tm_ds, t % p.st_tx, t / p.st_tx,
                             p.rparts + (p.rg_row0[b] + (long long)chunk * p.st_tiles + t) * kRegNV, sbase, bars);
      nbars = RgGeo<T>::RING;
      done = ctr + pk_ctr_rg(b);
    } else if (type == PK_SOLVE) {
      double D[kRedMaxNV], R[kRedMaxNV];
      const int olo = p.olo[b], ohi = min(p.cg.nz_global - 1, p.hi[b] + rz);
      const long long g0 = p.g_row0[b];
      pk_sum_rows(p.gparts, 3, g0, g0 + (long long)(ohi - olo + 1) * p.gram_tiles, s_red, D);
      const int h = p.hi[b] - p.lo[b] + 1;
      const long long r0 = p.rg_row0[b];
      pk_sum_rows(p.rparts, kRegNV, r0, r0 + (long long)((h + p.rg_c[b] - 1) / p.rg_c[b]) * p.st_tiles, s_red, R);
      if (threadIdx.x == 0) solve_one(p.solve, b, D, R, p.info + b * kInfoNV);
      done = ctr + pk_ctr_solve(b);
    } else if (type == PK_UPD) {
      const double* o = p.info + b * kInfoNV;
      const long long n = (long long)(p.hi[b] - p.lo[b] + 1) * p.cg.plane;
      const long long i0 = (long long)(sg.z + k) * p.upd_chunk, i1 = min(n, i0 + p.upd_chunk);
      const long long off = (long long)(p.lo[b] - p.frag_z0) * p.cg.plane;
      T* xb = p.xw + off;
      T* db = p.dmem + off;
      const T* gb = p.g + (long long)(p.lo[b] - p.rec_lo) * p.cg.plane;
      if (__ldcg(o + 8) != 0.0) {  // failed step: nothing applied (mirrors keep x current)
        if (p.mir.n > 0)
          for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) pk_mirror_store(p.mir, b, i, xb[i]);
      } else {
        const T cgc = (T)__ldcg(o + 10), cdc = (T)__ldcg(o + 11);
        auto upd1 = [&](long long i, T g, T d, T x) {
          T inc = mul_rn(-g, cgc);
          inc = add_rn(inc, mul_rn(d, cdc));
          const T xn = add_rn(x, inc);
          xb[i] = xn;
          if (p.mir.n > 0) pk_mirror_store(p.mir, b, i, xn);
          db[i] = inc;
        };
        using V = typename Vec16<T>::type;
        constexpr int VE = 16 / sizeof(T), UN = 4;
        const bool vec = ((i0 | i1 | off) % VE) == 0 && p.mir.n == 0 &&
                         (reinterpret_cast<uintptr_t>(xb) & 15) == 0 && (reinterpret_cast<uintptr_t>(gb) & 15) == 0;
        if (vec) {  // 16-byte accesses, UN vectors per thread in flight
          const long long nv = (i1 - i0) / VE;
          for (long long v0 = threadIdx.x; v0 < nv; v0 += (long long)blockDim.x * UN) {
            V gv[UN], dv[UN], xv[UN];
#pragma unroll
            for (int u = 0; u < UN; ++u) {
              const long long v = v0 + (long long)u * blockDim.x;
              if (v < nv) {
                const long long i = i0 + v * VE;
                gv[u] = __ldcg(reinterpret_cast<const V*>(gb + i));
                dv[u] = __ldcg(reinterpret_cast<const V*>(db + i));
                xv[u] = __ldcg(reinterpret_cast<const V*>(xb + i));
              }
            }
#pragma unroll
            for (int u = 0; u < UN; ++u) {
              const long long v = v0 + (long long)u * blockDim.x;
              if (v < nv) {
                const long long i = i0 + v * VE;
                const T* gs = reinterpret_cast<const T*>(&gv[u]);
                const T* ds = reinterpret_cast<const T*>(&dv[u]);
                const T* xs = reinterpret_cast<const T*>(&xv[u]);
                T xn[VE], inc[VE];
#pragma unroll
                for (int e = 0; e < VE; ++e) {
                  inc[e] = add_rn(mul_rn(-gs[e], cgc), mul_rn(ds[e], cdc));
                  xn[e] = add_rn(xs[e], inc[e]);
                }
                *reinterpret_cast<V*>(xb + i) = *reinterpret_cast<const V*>(xn);
                *reinterpret_cast<V*>(db + i) = *reinterpret_cast<const V*>(inc);
              }
            }
          }
        } else {
          for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) upd1(i, __ldcg(gb + i), __ldcg(db + i), __ldcg(xb + i));
        }
      }
      if (p.mir.n > 0) __threadfence_system();
    } else if (type == PK_RED) {
      double res[kRedMaxNV];
      if (sg.z == 0) {
        pk_sum_rows(p.eparts, kEvalNV, 0, (long long)p.nb * p.st_tiles, s_red, res);
        if (threadIdx.x == 0)
          for (int q = 0; q < kEvalNV; ++q) p.sums[1 + q] = res[q];
      } else {
        const long long b0 = (long long)(p.rec_lo - p.u_lo) * p.conv_tiles;
        pk_sum_rows(p.cparts, 1, b0, b0 + (long long)(p.rec_hi - p.rec_lo + 1) * p.conv_tiles, s_red, res);
        if (threadIdx.x == 0) p.sums[0] = res[0];
      }
      if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ctr + kPkCtrRed, 1) == 1) {  // the second reduction: finalise the recorder terms
          __threadfence();
          const double* sm = p.sums;
          const double data = 0.5 * __ldcg(sm), box = p.fin_eta * __ldcg(sm + 1), tv = p.fin_lam * __ldcg(sm + 2),
                       ax = p.fin_kappa * __ldcg(sm + 3);
          double* t = p.terms;
          t[0] = data; t[1] = box; t[2] = tv; t[3] = ax;
          t[4] = data + box + tv + ax;
          t[5] = __ldcg(sm + 4); t[6] = __ldcg(sm + 5);
        }
      }
    }

    // ---- completion --------------------------------------------------------
    __threadfence();
    fence_proxy_async_global();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 0; q < nbars; ++q) mbar_inval(&bars[q]);
      if (done) red_release_add(done, 1);
      if (p.trace) {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        p.trace[4ull * item + 2] = t_end;
      }
    }
  }
}

// launcher (sweep_pk.cu): `slots` receives the resident CTAs of the launch;
// nothing is launched while a.total == 0
cudaError_t pk_launch(const PkArgs<double>& a, int K, cudaStream_t s, int* slots);

}  // namespace bd3mg
