// Device helpers shared by the EDAA kernel translation units.
#pragma once
#include <cmath>
#include <cstdint>

#include "edaa_internal.cuh"

namespace edaa {
namespace dev {

constexpr int kExpTab = 256;  // entries of the exp_nonpos table (2^(i/256))

// Programmatic dependent launch: every kernel of the solve schedule is launched
// with programmatic stream serialization (launch_pdl); it lets its successor
// launch at once (launch_dependents at entry) and waits for its predecessor's
// completion and memory (griddep_wait) before its first global read, so kernel
// launch latency and per-CTA prologues overlap the previous kernel's tail.
// Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

__device__ __forceinline__ double log_floor() { return -69.07755278982137; }  // log(1e-30)

// D = A·B + D for one 8×8×4 fp64 tile. Lane (g = lane>>2, t = lane&3) holds
// A[g][t], B[t][g] and D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// SplitMix64 draw number `index` (0-based) of the stream seeded with `seed`:
// the state after index+1 increments (prng.hpp:15-26), mapped to [0,1)
// with the top 53 bits (prng.hpp:24-26).
__device__ __forceinline__ double splitmix_unit_at(uint64_t seed, uint64_t index) {
  uint64_t z = seed + (index + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return static_cast<double>(z >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ double max_like_std(double top, double s) {
  return (top < s) ? s : top;  // std::max(top, s): NaN in s is ignored
}

// Shared-memory plan of the pass kernel (one CTA per SM, two warp groups):
//   xs  nbuf × X tile          [Lpad][kXST] fp32/fp64  (tile i+2 loads while i, i+1 are used)
//   ws  W chunk (Y or Z)       [Lpad][WST]  fp64
//   ss  2 × projection/weights [QCpad][kSST] fp64 (band half 0; becomes the weights w)
//   sh  2 × projection half 1  [QCpad][kSST] fp64
//   st  2 × state tile         [QCpad][kNP] fp64 (A or logits of the chunk's columns)
//   gs  G blocks of the chunk's runs, then per-column and per-run scalars.
struct SmemLayout {
  int xs_off, xs_bytes, ws_off, ws_bytes, ss_off, sh_off, st_off, buf_bytes, st_bytes, gs_off, col_off,
      tab_off, slt_off, mbar_off, total;
};
constexpr int kNSB = 2;  // projection / weight tile buffers: P1(i) reuses w(i−2)'s after sfree

__host__ __device__ inline int align16(int b) { return (b + 15) & ~15; }

// W row stride (doubles) ≡ 2 mod 8: the P1 A-fragment reads rows 2 apart (band
// order of pass P1), 4·stride words ≡ 8 mod 32, so each half-warp's LDS.64 is one
// conflict-free wavefront.
__host__ __device__ inline int w_stride(int qcpad) { return qcpad + ((2 - qcpad % 8 + 8) % 8); }

// X tiles arrive by TMA with 128-byte swizzle: each smem row holds 128 bytes
// (32 floats, or 16 doubles — an fp64 tile is two 16-column halves).  Boxes
// are at most 256 rows, so L > 256 takes two row boxes of x_box_rows each.
__host__ __device__ inline int x_box_rows(const Dims& d) {
  return d.Lpad <= 256 ? d.Lpad : ((d.Lpad / 2 + 7) / 8) * 8;
}
__host__ __device__ inline int x_rows(const Dims& d) {
  const int br = x_box_rows(d);
  return ((d.Lpad + br - 1) / br) * br;
}
__host__ __device__ inline int x_tile_bytes(const Dims& d) {
  const int b = x_rows(d) * 128 * (d.xbytes / 4);
  return (b + 1023) & ~1023;
}
// Element offset of X[l][j] (0 ≤ j < 32) inside a swizzled tile buffer.
template <class XT>
__device__ __forceinline__ int xoff(int l, int j, int rows);
template <>
__device__ __forceinline__ int xoff<float>(int l, int j, int /*rows*/) {
  return l * 32 + ((((j >> 2) ^ (l & 7))) << 2) + (j & 3);
}
template <>
__device__ __forceinline__ int xoff<double>(int l, int j, int rows) {
  const int jj = j & 15;
  return (j >> 4) * rows * 16 + l * 16 + (((jj >> 1) ^ (l & 7)) << 1) + (jj & 1);
}

__host__ __device__ inline SmemLayout smem_layout(const Dims& d, int nbuf) {
  SmemLayout s;
  int off = 0;
  s.xs_off = off;  // TMA destination: 1024-byte aligned, 128-byte swizzled rows
  s.xs_bytes = x_tile_bytes(d);
  off += nbuf * s.xs_bytes;
  s.ws_off = off;  // 2 W chunks: the current one and the next item's, prefetched by cp.async
  s.ws_bytes = align16(d.Lpad * w_stride(d.QCpad) * 8);
  off += d.nwb * s.ws_bytes;
  s.buf_bytes = align16(d.QCpad * kSST * 8);
  s.ss_off = off;  // nsb buffers of projection half 0 / weights
  off += kNSB * s.buf_bytes;
  s.sh_off = off;  // nsb buffers of projection half 1
  off += kNSB * s.buf_bytes;
  s.st_bytes = align16(d.QCpad * kNP * 8);
  s.st_off = off;
  off += 3 * s.st_bytes;  // state tiles i, i+1, i+2 in flight
  s.gs_off = off;
  off += align16(d.RC * d.p * d.p * 8);
  // m_run, S_run, colm, collogS, eta (QCpad each), fac[2][QCpad]; obj_run (RC), hobj (4·RC)
  s.col_off = off;
  off += align16((7 * d.QCpad + 5 * d.RC) * 8);
  s.tab_off = off;  // 2^(i/256) table of exp_nonpos
  off += kExpTab * 8;
  s.slt_off = off;  // first tile of every pixel slice (nslices + 1 ints)
  off += align16((d.nslices + 1) * 4);
  s.mbar_off = off;  // full[4], empty[4] X ring; sready[2], wready[2] hand-offs; sfree[4]
  off += 16 * 8;
  s.total = off;
  return s;
}


// ---- exp for non-positive arguments (softmax weights), ~1 ulp -------------------
// x = (k/256)·ln2 + r, |r| ≤ ln2/512:  e^x = 2^⌊k/256⌋ · 2^{(k mod 256)/256} · e^r.
// k = round(x·256/ln2) by the 1.5·2^52 shifter (one FMA; k is the low word), the
// 256 table entries correctly rounded (70-digit decimal arithmetic), a Cody–Waite
// split of ln2/256 (hi has 33 significant bits: k·hi exact for |k| < 2^19), a
// degree-5 Taylor polynomial (truncation < 1e-20) and the 2^⌊k/256⌋ scale added
// to the exponent field with an integer add.  10 fp64-pipe instructions on the
// dependent chain, against ~20 for libdevice exp: these scalar fp64 ops share the
// pipe with the DMMA contractions and sit on the per-pixel update's critical path.
// In global memory, not __constant__: every thread loads a different entry, which the
// constant cache would serialise (measured ~4k cycles of pass-kernel prologue).
__device__ const double kExp2Tab[kExpTab] = {
    1.0, 1.0027112750502025, 1.0054299011128027, 1.0081558981184175,
    1.0108892860517005, 1.0136300849514894, 1.016378314910953, 1.019133996077738,
    1.0218971486541166, 1.0246677928971357, 1.0274459491187637, 1.030231637686041,
    1.0330248790212284, 1.0358256936019572, 1.0386341019613787, 1.041450124688316,
    1.0442737824274138, 1.0471050958792898, 1.0499440858006872, 1.0527907730046264,
    1.0556451783605572, 1.0585073227945128, 1.061377227289262, 1.0642549128844645,
    1.0671404006768237, 1.0700337118202419, 1.0729348675259756, 1.075843889062791,
    1.0787607977571199, 1.0816856149932152, 1.0846183622133092, 1.0875590609177697,
    1.0905077326652577, 1.0934643990728858, 1.0964290818163769, 1.099401802630222,
    1.102382583307841, 1.1053714457017412, 1.1083684117236787, 1.1113735033448175,
    1.1143867425958924, 1.1174081515673693, 1.1204377524096067, 1.12347556733302,
    1.1265216186082418, 1.129575928566288, 1.1326385195987192, 1.1357094141578055,
    1.1387886347566916, 1.1418762039695616, 1.1449721444318042, 1.148076478840179,
    1.1511892299529827, 1.154310420590216, 1.1574400736337511, 1.1605782120274988,
    1.1637248587775775, 1.1668800369524817, 1.1700437696832502, 1.1732160801636373,
    1.1763969916502812, 1.1795865274628758, 1.182784710984341, 1.1859915656609938,
    1.189207115002721, 1.1924313825831512, 1.1956643920398273, 1.1989061670743806,
    1.202156731452703, 1.2054161090051239, 1.2086843236265816, 1.2119613992768012,
    1.215247359980469, 1.2185422298274085, 1.2218460329727576, 1.2251587936371455,
    1.22848053610687, 1.2318112847340759, 1.2351510639369334, 1.2384998981998165,
    1.241857812073484, 1.245224830175258, 1.2486009771892048, 1.2519862778663162,
    1.255380757024691, 1.2587844395497165, 1.2621973503942507, 1.2656195145788063,
    1.2690509571917332, 1.2724917033894028, 1.275941778396392, 1.2794012075056693,
    1.2828700160787783, 1.2863482295460256, 1.2898358734066657, 1.2933329732290895,
    1.2968395546510096, 1.3003556433796506, 1.3038812651919358, 1.3074164459346773,
    1.3109612115247644, 1.3145155879493546, 1.318079601266064, 1.3216532776031575,
    1.3252366431597413, 1.3288297242059544, 1.3324325470831615, 1.3360451382041458,
    1.339667524053303, 1.3432997311868353, 1.3469417862329458, 1.3505937158920345,
    1.3542555469368927, 1.3579273062129011, 1.3616090206382248, 1.365300717204012,
    1.3690024229745905, 1.3727141650876684, 1.3764359707545302, 1.380167867260238,
    1.383909881963832, 1.387662042298529, 1.3914243757719262, 1.3951969099662003,
    1.3989796725383112, 1.4027726912202048, 1.4065759938190154, 1.4103896082172707,
    1.4142135623730951, 1.4180478843204152, 1.4218926021691656, 1.4257477441054942,
    1.42961333839197, 1.433489413367789, 1.4373759974489824, 1.4412731191286257,
    1.4451808069770467, 1.449099089642035, 1.4530279958490526, 1.4569675544014438,
    1.460917794180647, 1.4648787441464057, 1.4688504333369818, 1.4728328908693675,
    1.4768261459394993, 1.4808302278224719, 1.4848451658727524, 1.488870989524397,
    1.4929077282912648, 1.4969554117672355, 1.5010140696264256, 1.5050837316234065,
    1.5091644275934228, 1.5132561874526098, 1.5173590411982147, 1.5214730189088146,
    1.5255981507445384, 1.529734466947287, 1.533881997840956, 1.5380407738316568,
    1.5422108254079407, 1.5463921831410214, 1.550584877685, 1.5547889397770887,
    1.559004400237837, 1.5632312899713576, 1.567469639965553, 1.5717194812923414,
    1.5759808451078865, 1.5802537626528246, 1.5845382652524937, 1.588834384317164,
    1.593142151342267, 1.597461597908627, 1.6017927556826934, 1.606135656416771,
    1.6104903319492543, 1.6148568142048607, 1.6192351351948637, 1.6236253270173289,
    1.6280274218573478, 1.632441451987275, 1.6368674497669644, 1.6413054476440063,
    1.645755478153965, 1.6502175739206177, 1.6546917676561943, 1.6591780921616162,
    1.6636765803267364, 1.6681872651305825, 1.6727101796415966, 1.6772453570178785,
    1.681792830507429, 1.6863526334483934, 1.6909247992693053, 1.6955093614893326,
    1.7001063537185235, 1.7047158096580513, 1.709337763100463, 1.713972247929926,
    1.718619298122478, 1.723278947746274, 1.7279512309618377, 1.732636182022311,
    1.7373338352737062, 1.7420442251551564, 1.746767386199169, 1.7515033530318782,
    1.7562521603732995, 1.761013843037584, 1.7657884359332727, 1.7705759740635547,
    1.7753764925265212, 1.7801900265154245, 1.785016611318935, 1.789856282321401,
    1.7947090750031072, 1.7995750249405351, 1.804454167806624, 1.809346539371032,
    1.8142521755003989, 1.8191711121586085, 1.8241033854070534, 1.8290490314048973,
    1.8340080864093424, 1.8389805867758937, 1.843966568958626, 1.8489660695104508,
    1.8539791250833855, 1.8590057724288205, 1.864046048397789, 1.8690999899412386,
    1.8741676341103, 1.8792490180565602, 1.8843441790323345, 1.8894531543909392,
    1.8945759815869656, 1.8997126981765553, 1.9048633418176741, 1.9100279502703899,
    1.9152065613971474, 1.9203992131630474, 1.925605943636125, 1.930826790987627,
    1.9360617934922943, 1.9413109895286405, 1.9465744175792332, 1.9518521162309783,
    1.9571441241754002, 1.9624504802089273, 1.9677712232331759, 1.9731063922552343,
    1.978456026387951, 1.9838201648502194, 1.9891988469672663, 1.9945921121709402,
};

__device__ __forceinline__ void load_exp_table(double* T, int tid) {
  for (int i = tid; i < kExpTab; i += blockDim.x) T[i] = kExp2Tab[i];
}

__device__ __forceinline__ double exp_nonpos(double x, const double* T) {
  // Branch-free: x ≤ −745 (incl. −inf) → 0, NaN → NaN by the final select; the
  // 2^⌊k/256⌋ scale is split over two normal powers of two so denormal results
  // (−745 < x < −708) round once, as std::exp's do.
  const double t = fma(x, 369.3299304675746, 6755399441055744.0);  // 256/ln2, 1.5·2^52
  const double kd = t - 6755399441055744.0;
  const int k = __double2loint(t);
  double r = fma(kd, -0.0027076061742263846, x);  // ln2/256, high part
  r = fma(kd, 1.6409824502660487e-13, r);         // ln2/256, low part
  double q = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = fma(q, r, 1.0);
  const int e = k >> 8;  // floor(k / 256)
  const int e1 = e >> 1, e2 = e - e1;
  const double ts = T[k & (kExpTab - 1)] * __hiloint2double((e1 + 1023) << 20, 0);  // off the chain
  const double y = (q * ts) * __hiloint2double((e2 + 1023) << 20, 0);
  return (x > -745.0) ? y : ((x == x) ? 0.0 : x);
}


// ---- mbarrier + TMA (cp.async.bulk.tensor) ----------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait2() { asm volatile("cp.async.wait_group 2;\n" ::: "memory"); }

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace dev
}  // namespace edaa
