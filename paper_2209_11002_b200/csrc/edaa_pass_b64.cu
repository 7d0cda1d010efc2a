// B pass with 64-pixel LOGICAL tiles (fp32 image): the same arithmetic as k_pass<kModeB>, one
// hand-off per two 32-pixel X slots.
//
// Why (profiles/round2/EXPERIMENTS.md §7): a band sweep shows the contraction loops of k_pass at
// ~95% of the DMMA roof and a FIXED ≈ 4.5k cycles per 32-pixel tile around them — mbarrier
// round trips between the MMA and update groups, S stores, rescale, bookkeeping, DMMA pipe
// fill and drain at the two phase boundaries.  Per pixel that cost halves when one hand-off
// covers 64 pixels.  Shared memory (227 KB) then holds, at L = 198: 5 X slots of 32 pixels
// (128 KB; P3 releases its first slot half-way so the ring stays one slot short of three
// logical tiles), ONE W chunk buffer (41.6 KB), the S / w tiles without the band-half split
// (P1 = 8 pixel groups × all bands: 2 × 13 KB) and no state tiles (the logits come from global
// memory into registers).  It fits for L ≤ 232 with a 24-column chunk (cfg0–cfg4); other shapes
// and fp64 images keep k_pass.
//
// Partial sums: P3 accumulates the same 32-pixel k-step sequence per slice as k_pass (two
// slots in order = two tiles in order) and flushes per (slice, chunk) item, so Y is bitwise
// what k_pass produces; P1's g = XᵀZ is ONE band-ascending DMMA chain per (pixel, column)
// here against two half-band chains added in k_pass — equal to rounding, and the choice
// between the kernels depends on (L, p, image type) only, never on the batch.
#include "edaa_pass.cuh"

namespace edaa {
namespace pass_impl {

constexpr int kNP2 = 2 * kNP;     // pixels per logical tile
constexpr int kSST2 = kNP2 + 4;   // S / w tile row stride (doubles): ≡ 8 words mod 32 like kSST
constexpr int kMaxRing = 8;

struct Lay64 {
  int xs_off, xs_bytes, ws_off, ws_bytes, ss_off, buf_bytes, col_off, tab_off, slt_off, mbar_off, total;
};

// nbuf X slots (32 pixels each), one W chunk, kNSB S/w tiles [QCpad][kSST2].  No state tiles: the
// update reads its logits straight from global memory into registers ahead of the wait for S(i)
// (measured equal to a cp.async state ring at cfg1 / cfg2, and it is what lets L = 224 fit).
__host__ __device__ inline Lay64 layout_b64(const Dims& d, int nbuf) {
  Lay64 s;
  int off = 0;
  s.xs_off = off;
  s.xs_bytes = x_tile_bytes(d);
  off += nbuf * s.xs_bytes;
  s.ws_off = off;
  s.ws_bytes = align16(d.Lpad * w_stride(d.QCpad) * 8);
  off += s.ws_bytes;
  s.buf_bytes = align16(d.QCpad * kSST2 * 8);
  s.ss_off = off;
  off += kNSB * s.buf_bytes;
  s.col_off = off;  // m_run, S_run, c_m, c_eta (QCpad each), fac[2][QCpad]
  off += align16(6 * d.QCpad * 8);
  s.tab_off = off;
  off += kExpTab * 8;
  s.slt_off = off;
  off += align16((d.nslices + 1) * 4);
  s.mbar_off = off;  // full[8], empty[8], sready[2], wready[2], sfree[2]
  off += (2 * kMaxRing + 6) * 8;
  s.total = off;
  return s;
}

// P3 over ONE 32-pixel slot: C[l][c] += Σ_j X[l][j]·w[c][j]; w points at the slot's first pixel column.
template <int R, int CT, int RTW>
__device__ __forceinline__ void accumulate_slot(double (&ac)[RTW][kMaxCT][2], const float* xs, const double* w,
                                                int gwarp, int g, int t4, const int (&xo)[kNP / 4]) {
  const double* wrow = w + g * kSST2 + t4;
#pragma unroll
  for (int kk = 0; kk < kNP / 4; ++kk) {
    double bw[CT];
#pragma unroll
    for (int ct = 0; ct < CT; ++ct) bw[ct] = wrow[ct * 8 * kSST2 + kk * 4];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const double ax = static_cast<double>(xs[(gwarp + 8 * i) * 8 * kXRow<float> + xo[kk]]);
#pragma unroll
      for (int ct = 0; ct < CT; ++ct) dmma(ac[i][ct], ax, bw[ct]);
    }
  }
}

template <int RTW, int CTF, bool ILV>
__global__ void __launch_bounds__(kThreads, 1) k_pass_b64(PassArgs pa, const __grid_constant__ CUtensorMap xmap,
                                                          int nbuf) {
  extern __shared__ __align__(16) unsigned char smem[];
  using XT = float;
  const Dims& d = pa.d;
  const Lay64 lay = layout_b64(d, nbuf);
  double* ws = reinterpret_cast<double*>(smem + lay.ws_off);
  int* slt = reinterpret_cast<int*>(smem + lay.slt_off);
  double* m_run = reinterpret_cast<double*>(smem + lay.col_off);
  double* S_run = m_run + kQMax;
  double* c_m = S_run + kQMax;    // normaliser max + log-sum of the previous logits
  double* c_eta = c_m + kQMax;    // η_b of the column's run
  double* facb = c_eta + kQMax;   // [2][QCpad] running-max rescale of logical tile i % 2
  double* etab = reinterpret_cast<double*>(smem + lay.tab_off);
  auto xslot = [&](int b) { return reinterpret_cast<XT*>(smem + lay.xs_off + b * lay.xs_bytes); };
  auto sbuf = [&](int i) { return reinterpret_cast<double*>(smem + lay.ss_off + (i & 1) * lay.buf_bytes); };

  const int tid = threadIdx.x;
  const bool mma_group = tid < kGroup;
  const int gtid = tid & (kGroup - 1);
  const int lane = tid & 31, gwarp = gtid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int p = d.p;
  const int nRT = d.Lpad / 8;
  const int WST = w_stride(kQMax);

  const int K = d.NCH * (d.sl1 - d.sl0);
  const int item_begin = static_cast<int>((static_cast<long long>(blockIdx.x) * K) / gridDim.x);
  const int item_end = static_cast<int>((static_cast<long long>(blockIdx.x + 1) * K) / gridDim.x);
  int ntile = 0;  // 32-pixel tiles (X slots) of this CTA; even: slices are tile pairs
  for (int k = item_begin; k < item_end; ++k) {
    const int s = item_slice_t<ILV>(d, k);
    ntile += slice_tile(d, s + 1) - slice_tile(d, s);
  }
  if (ntile == 0) return;
  const int nlt = ntile / 2;  // logical tiles

  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + lay.mbar_off);
  unsigned long long* empty = full + kMaxRing;
  unsigned long long* sready = empty + kMaxRing;
  unsigned long long* wready = sready + 2;
  unsigned long long* sfree = wready + 2;
  for (int i = tid; i <= d.nslices; i += kThreads) slt[i] = slice_tile(d, i);
  if (tid == 0) {
    for (int b = 0; b < nbuf; ++b) {
      mbar_init(full + b, 1);
      mbar_init(empty + b, 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(sready + b, 8);
      mbar_init(wready + b, 8);
      mbar_init(sfree + b, 8);
    }
    mbar_fence_init();
  }
  auto warp_arrive = [&](unsigned long long* bar) {
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
  };
  if (tid < kQMax) facb[tid] = facb[kQMax + tid] = 1.0;
  griddep_launch_dependents();
  griddep_wait();
  __syncthreads();

  if (mma_group) {
    // =========================== MMA group ===========================
    double acc[RTW][kMaxCT][2];
#pragma unroll
    for (int i = 0; i < RTW; ++i)
#pragma unroll
      for (int c = 0; c < kMaxCT; ++c) acc[i][c][0] = acc[i][c][1] = 0.0;
    const int my_rt = (nRT - gwarp + 7) / 8;  // row tiles gwarp + 8·i < nRT
    Cursor xc, p1c, p3c;  // 32-pixel tile cursors: X producer, P1 (two per logical tile), P3
    cursor_set_t<ILV>(xc, d, slt, item_begin);
    cursor_set_t<ILV>(p1c, d, slt, item_begin);
    cursor_set_t<ILV>(p3c, d, slt, item_begin);
    int wchunk = -1;
    auto w_fetch = [&](int chunk) {
      constexpr int kV = kQMax / 2;
      for (int e = gtid; e < d.Lpad * kV; e += kGroup) {
        const int l = e / kV, c2 = e - l * kV;
        cp_async16(ws + l * WST + 2 * c2, pa.W + static_cast<size_t>(l) * d.Qs + chunk * kQMax + 2 * c2);
      }
      cp_async_commit();
    };
    const int xrows = x_rows(d), brows = x_box_rows(d);
    int xo3[kNP / 4];
#pragma unroll
    for (int kk = 0; kk < kNP / 4; ++kk) xo3[kk] = xoff<XT>(g, kk * 4 + t4, xrows);
    // P1 unit of the warp: slot half h of the logical tile, 8 pixels pt of that slot, ALL bands.
    const int p1_h = gwarp >> 2, p1_pt = gwarp & 3;
    const int p1_xo0 = xoff<XT>(2 * t4, p1_pt * 8 + g, xrows), p1_xo1 = xoff<XT>(2 * t4 + 1, p1_pt * 8 + g, xrows);
    const int p1_mn = d.Lpad / 8;
    const int nbox = xrows / brows;
    const unsigned tile_tx = static_cast<unsigned>(nbox * brows * 128);
    // X slot of 32-pixel tile t of this CTA's stream: slot t % nbuf, completion t / nbuf.
    auto load_slot = [&](int t) {  // producer (MMA thread 0); every MMA thread advances the cursor
      if (gtid == 0) {
        const int b = t % nbuf, q = t / nbuf;
        if (q > 0) mbar_wait(empty + b, (q - 1) & 1);  // the slot's previous tile released by all 8 MMA warps
        mbar_expect_tx(full + b, tile_tx);
        XT* dst = xslot(b);
        for (int bx = 0; bx < nbox; ++bx) tma_load_2d(dst + bx * brows * 32, &xmap, xc.tile * kNP, bx * brows, full + b);
      }
      cursor_next_t<ILV>(xc, d, slt);
    };
    auto slot_wait = [&](int t) {
      mbar_wait(full + t % nbuf, (t / nbuf) & 1);
      return t % nbuf;
    };
    auto slot_release = [&](int t) {
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + t % nbuf);
    };
    // P1 of logical tile i: S[c][j] = Σ_l W[l][c]·X[l][j] for the warp's 8 pixels of its slot, all bands.
    auto phase1 = [&](int i) {
      if (i >= kNSB) mbar_wait(sfree + (i & 1), ((i >> 1) - 1) & 1);  // w(i−2) consumed by P3(i−2)
      const int chunk = p1c.chunk;
      if (chunk != wchunk) {  // one W buffer: restage once every MMA warp is past its previous P1
        if (wchunk >= 0) {
          bar_sync(bars::kMma, kGroup);
          w_fetch(chunk);
        }
        cp_async_wait0();
        bar_sync(bars::kMma, kGroup);
        wchunk = chunk;
      }
      const XT* xs = xslot(slot_wait(2 * i + p1_h));
      double c1[CTF][2];
#pragma unroll
      for (int c = 0; c < CTF; ++c) c1[c][0] = c1[c][1] = 0.0;
      const double* wcol = ws + 2 * t4 * WST + g;
#pragma unroll kP1Unroll
      for (int m = 0; m < p1_mn; ++m) {
        const XT* xr = xs + m * 8 * kXRow<XT>;
        const double bx0 = static_cast<double>(xr[p1_xo0]);
        const double bx1 = static_cast<double>(xr[p1_xo1]);
        const double* w0 = wcol + m * 8 * WST;
        const double* w1 = w0 + WST;
#pragma unroll
        for (int ct = 0; ct < CTF; ++ct) dmma(c1[ct], w0[ct * 8], bx0);
#pragma unroll
        for (int ct = 0; ct < CTF; ++ct) dmma(c1[ct], w1[ct * 8], bx1);
      }
      double* dst = sbuf(i);
#pragma unroll
      for (int ct = 0; ct < CTF; ++ct)
        *reinterpret_cast<double2*>(dst + (ct * 8 + g) * kSST2 + p1_h * kNP + p1_pt * 8 + 2 * t4) =
            make_double2(c1[ct][0], c1[ct][1]);
      cursor_next_t<ILV>(p1c, d, slt);
      cursor_next_t<ILV>(p1c, d, slt);
      warp_arrive(sready + (i & 1));
    };
    auto p3_slot = [&](const XT* xs, const double* w) {
      switch (my_rt) {  // warp-uniform: the DMMAs below are unpredicated
        case 1: accumulate_slot<1, CTF>(acc, xs, w, gwarp, g, t4, xo3); break;
        case 2: accumulate_slot<2, CTF>(acc, xs, w, gwarp, g, t4, xo3); break;
        case 3: accumulate_slot<3, CTF>(acc, xs, w, gwarp, g, t4, xo3); break;
        case 4: if constexpr (RTW >= 4) accumulate_slot<4, CTF>(acc, xs, w, gwarp, g, t4, xo3); break;
        case 5: if constexpr (RTW >= 5) accumulate_slot<5, CTF>(acc, xs, w, gwarp, g, t4, xo3); break;
        case 6: if constexpr (RTW >= 6) accumulate_slot<6, CTF>(acc, xs, w, gwarp, g, t4, xo3); break;
        default: break;
      }
    };

    w_fetch(item_chunk_t<ILV>(d, item_begin));                    // the first W chunk …
    for (int t = 0; t < nbuf && t < ntile; ++t) load_slot(t);    // … and every ring slot in flight
    cp_async_wait0();
    bar_sync(bars::kMma, kGroup);
    wchunk = item_chunk_t<ILV>(d, item_begin);
    phase1(0);
    for (int it = 0; it < nlt; ++it) {
      // slot 2it + nbuf − 1 into the slot P3(it − 1) released last
      if (2 * it + nbuf - 1 < ntile && it > 0) load_slot(2 * it + nbuf - 1);
      if (it + 1 < nlt) phase1(it + 1);
      mbar_wait(wready + (it & 1), (it >> 1) & 1);  // w(it), fac(it) ready
      {
        const double* fac = facb + (it & 1) * kQMax;
#pragma unroll
        for (int ct = 0; ct < kMaxCT; ++ct) {
          const double f0 = fac[ct * 8 + 2 * t4], f1 = fac[ct * 8 + 2 * t4 + 1];
          if (f0 != 1.0 || f1 != 1.0) {
#pragma unroll
            for (int i = 0; i < RTW; ++i) {
              acc[i][ct][0] *= f0;
              acc[i][ct][1] *= f1;
            }
          }
        }
      }
      const double* w = sbuf(it);
      p3_slot(xslot(slot_wait(2 * it)), w);
      slot_release(2 * it);
      // the slot just released takes tile 2it + nbuf (one slot short of three logical tiles in the ring)
      if (2 * it + nbuf < ntile) load_slot(2 * it + nbuf);
      p3_slot(xslot(slot_wait(2 * it + 1)), w + kNP);
      if (p3c.tile + 2 == p3c.tend) {  // the item's last logical tile: flush and restart its partials
        const int slice = p3c.slice, col0 = p3c.chunk * kQMax;
#pragma unroll
        for (int i = 0; i < RTW; ++i) {
          const int rt = gwarp + 8 * i;
          if (rt < nRT) {
            const int row = rt * 8 + g;
#pragma unroll
            for (int ct = 0; ct < kMaxCT; ++ct) {
              double* dst = pa.part_C + (static_cast<size_t>(slice) * d.Lrows + row) * d.Qs + col0 + ct * 8 + 2 * t4;
              *reinterpret_cast<double2*>(dst) = make_double2(acc[i][ct][0], acc[i][ct][1]);
            }
          }
#pragma unroll
          for (int ct = 0; ct < kMaxCT; ++ct) acc[i][ct][0] = acc[i][ct][1] = 0.0;
        }
      }
      slot_release(2 * it + 1);
      warp_arrive(sfree + (it & 1));
      cursor_next_t<ILV>(p3c, d, slt);
      cursor_next_t<ILV>(p3c, d, slt);
    }
  } else {
    // ========================== update group ==========================
    // the exp table is this group's alone: loaded here, off the MMA group's path to its first tile
    // (the bar_sync at the top of the loop orders it before the first exp)
    if (gtid < kExpTab) etab[gtid] = kExp2Tab[gtid];
    Cursor p2c;
    cursor_set_t<ILV>(p2c, d, slt, item_begin);
    int cchunk = -1;
    for (int it = 0; it < nlt; ++it) {
      const ChunkInfo ci = chunk_info(d, p2c.chunk);
      const int j0 = p2c.tile * kNP;
      const bool item_first = p2c.tile == p2c.tstart;
      const bool item_last = p2c.tile + 2 == p2c.tend;
      bar_sync(bars::kUpd, kGroup);  // everyone is done with the previous tile's and item's scalars
      if (ci.chunk != cchunk) {
        if (gtid < kQMax) {
          const int c = gtid;
          const bool real = c < ci.ncol;
          c_m[c] = real ? pa.colm[ci.col0 + c] + pa.collogS[ci.col0 + c] : 0.0;  // log b_old = ℓ − (m + log S)
          c_eta[c] = real ? pa.eta_b[ci.run0 + c / p] : 0.0;
        }
        cchunk = ci.chunk;
      }
      if (item_first && gtid < kQMax) {
        m_run[gtid] = -INFINITY;
        S_run[gtid] = 0.0;
      }
      constexpr int PPL = kNP2 / 8;
      const int uc = gtid >> 3, ul8 = gtid & 7;  // 8 lanes per column, 8 pixels per lane (j = k·8 + l8)
      double lg[PPL];  // the lane's 8 logits, in flight across the barrier and the wait for S(i)
#pragma unroll
      for (int k = 0; k < PPL; ++k) {
        const int pix = j0 + k * 8 + ul8;
        lg[k] = (uc < ci.ncol && pix < d.N) ? pa.Lg[static_cast<size_t>(ci.srow0 + uc) * d.Npad + pix] : 0.0;
      }
      bar_sync(bars::kUpd, kGroup);
      mbar_wait(sready + (it & 1), (it >> 1) & 1);  // S(i) ready
      if (pa.dbg & 256) {  // development (EDAA_DBG=256, as in k_pass): bare hand-shake, no update work
        warp_arrive(wready + (it & 1));
        cursor_next_t<ILV>(p2c, d, slt);
        cursor_next_t<ILV>(p2c, d, slt);
        continue;
      }
      double* ss = sbuf(it);
      double* fac = facb + (it & 1) * kQMax;
      {
        // new logits
        const int c = uc, l8 = ul8;
        const bool active = c < kQMax;
        double ell[PPL];
        double tmax = -INFINITY;
        if (active) {
          const bool real = c < ci.ncol;
#pragma unroll
          for (int k = 0; k < PPL; ++k) {
            const int j = k * 8 + l8, pix = j0 + j;
            double v = -INFINITY;
            if (real && pix < d.N) {
              double lb = lg[k] - c_m[c];                           // log b_old
              lb = (lb < log_floor()) ? log_floor() : lb;           // log max(b, 1e-30)
              v = lb + ss[c * kSST2 + j] * c_eta[c];                // + η_b·(−∇_B)
              pa.Lg[static_cast<size_t>(ci.srow0 + c) * d.Npad + pix] = v;
            }
            ell[k] = v;
            tmax = fmax(tmax, v);
          }
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        double tsum = 0.0, mn = -INFINITY, mo = -INFINITY;
        if (active) {
          mo = m_run[c];
          mn = fmax(mo, tmax);
#pragma unroll
          for (int k = 0; k < PPL; ++k) {
            const double w = (pa.dbg & 2) ? 1.0 : ((mn == -INFINITY) ? 0.0 : exp_nonpos(ell[k] - mn, etab));
            ss[c * kSST2 + k * 8 + l8] = w;
            tsum += w;
          }
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
        if (active && l8 == 0) {
          const double f = (mn == -INFINITY || mn == mo) ? 1.0 : exp_nonpos(mo - mn, etab);
          fac[c] = f;
          S_run[c] = S_run[c] * f + tsum;
          m_run[c] = mn;
        }
      }
      if (item_last) {
        bar_sync(bars::kUpd, kGroup);
        if (gtid < kQMax) {
          pa.part_m[static_cast<size_t>(p2c.slice) * d.Qs + ci.col0 + gtid] = m_run[gtid];
          pa.part_S[static_cast<size_t>(p2c.slice) * d.Qs + ci.col0 + gtid] = S_run[gtid];
        }
      }
      warp_arrive(wready + (it & 1));
      cursor_next_t<ILV>(p2c, d, slt);
      cursor_next_t<ILV>(p2c, d, slt);
    }
  }
}

template <int RTW, int CTF>
cudaError_t launch_b64_ctf(const PassArgs& a, cudaStream_t st) {
  const dim3 grid(std::min(a.d.NCH * (a.d.sl1 - a.d.sl0), a.d.ncta));
  const size_t smem = layout_b64(a.d, a.d.nbuf64).total;
  void (*kern)(PassArgs, CUtensorMap, int) = a.d.ilv ? k_pass_b64<RTW, CTF, true> : k_pass_b64<RTW, CTF, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(a.d.pdl != 0, kern, grid, dim3(kThreads), smem, st, a, *static_cast<const CUtensorMap*>(a.xmap),
                 a.d.nbuf64);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace pass_impl

size_t pass_b64_smem_bytes(const Dims& d, int nbuf) { return pass_impl::layout_b64(d, nbuf).total; }

cudaError_t launch_pass_b64(const PassArgs& a, cudaStream_t st) {
  const bool wide = (a.d.Lpad / 8 + kQMax / 8) > 32;  // k_pass's RTW rule
  const bool one = a.d.NCH == 1 && a.d.M * a.d.p <= 8;
  if (wide) return one ? pass_impl::launch_b64_ctf<6, 1>(a, st) : pass_impl::launch_b64_ctf<6, kMaxCT>(a, st);
  return one ? pass_impl::launch_b64_ctf<4, 1>(a, st) : pass_impl::launch_b64_ctf<4, kMaxCT>(a, st);
}

}  // namespace edaa
