// nlm_sym.cuh -- NLM variant "sym_tmem": the offset-symmetric formulation.  (NLM is not in
// PAPER.md; definition DESIGN.md R11-R14, this formulation R30.)
//
// With the boundary-extended image u_B, the patch distance is symmetric under a shift:
//   d_{-o}(p) = sum_t (u_B(p+t) - u_B(p+t-o))^2 = d_o(p-o)          (substitute t' = t - o)
// so one weight w_o(q) = 2^(-coef * d_o(q)) serves two (pixel, offset) pairs:
//   own      (q, o):   num(q)   += w * u_B(q+o),  den(q)   += w
//   partner  (q+o,-o): num(q+o) += w * u_B(q),    den(q+o) += w
// Walking the half set  O+ = {oy > 0, |ox| <= S} u {oy = 0, 0 < ox <= S}  (plus the centre,
// w = 1) covers every pair of the (2S+1)^2 window exactly once, with half the patch distances
// and half the ex2 of the direct enumeration.
//
// Layout (one warp = one 4-column-per-lane strip of 128 d-columns, walking 32 rows):
//   * the CTA's image tile (plus the 2(S+P)+1 halo rows and 2S+2P halo columns, boundary
//     applied at load time) sits in shared memory; 4 warps stack vertically (128 output rows);
//   * a warp's d-columns are [X-S, X-S+128): the 128-2S output columns plus S on each side,
//     the partner sources tile - o of the shifts that cross the strip edge;
//   * per search row oy (outer loop) the warp walks d-rows y from -oy to 31 (the rows above
//     the strip are partner sources), the vertical patch sum sliding
//        d(y) = d(y-1) + H(y+P) - H(y-P-1),  H(r) = horizontal patch sum of (u(q)-u(q+o))^2,
//     in registers for all 2S+1 ox at once, as float2 pairs of adjacent ox (FADD2/FFMA2);
//     the second offset of a pair is evaluated ONE COLUMN TO THE LEFT ("b lags"): for the pair
//     (ox, ox+1) lane column k holds (d_(ox)(k), d_(ox+1)(k-1)), so both halves read the same
//     shifted sample u(k + ox + t) (a broadcast operand) and the same u(q + o) = u(k + ox), and
//     send their partner contributions to the same column k + ox; only the shared centre window
//     is read as the pair (c(t), c(t-1)).  No per-pair register-pair assembly (MOV) is left;
//     the own sums of column k then collect half a of k and half b of k+1 (one shuffle for k=3);
//     H_old is recomputed from the image rows, not stored (no ring);
//   * own contributions accumulate in registers per row; partner contributions accumulate in a
//     (4+2S)-column register window which the lanes exchange by warp shuffles (columns that
//     belong to the neighbouring lanes);
//   * num/den of the warp's 32 x 128 pixels live in TENSOR MEMORY (one TMEM lane per thread,
//     8 columns per row: num[4], den[4]), read-modify-written once per (row, oy) for the own
//     row and once for the partner row, with tcgen05.ld / tcgen05.st -- the on-chip space that
//     lets the walk be long (32 rows) without giving up registers or shared memory.
//   * interior tiles are staged by 8-byte cp.async (all in flight), border tiles through read_B;
//     a barrier after each pass keeps the CTA's warps on one pass body (instruction fetch).
// Variants: "sym_tmem" (2 CTAs x 4 warps per SM, the default for large calls), "sym_ring" (RING:
// one CTA/SM whose TMEM also holds the last 2P+1 H rows, so a step computes only the entering
// row), "sym_tmem8" (NW = 8: one 8-warp CTA per SM).  DESIGN.md §5 has the measurements.
// Results agree with the direct definition to rounding (tolerance-checked, R16).
#pragma once

#include "nlm_common.cuh"

namespace icl {

__device__ __forceinline__ float2 s2_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 s2_sub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 s2_mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 s2_fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// ---- tensor memory (tcgen05) helpers: 32 lanes x 32 bit, 8 consecutive columns per thread
__device__ __forceinline__ void tm_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r0, r1, r2, r3, r4, r5, r6, r7;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(r4), "=r"(r5), "=r"(r6), "=r"(r7)
               : "r"(taddr));
  v[0] = __uint_as_float(r0); v[1] = __uint_as_float(r1); v[2] = __uint_as_float(r2); v[3] = __uint_as_float(r3);
  v[4] = __uint_as_float(r4); v[5] = __uint_as_float(r5); v[6] = __uint_as_float(r6); v[7] = __uint_as_float(r7);
}
// wait for the outstanding tcgen05.ld (tm_wait_ld), then pin the loaded values behind it (tm_pin8):
// no use of them can be scheduled above the wait
__device__ __forceinline__ void tm_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// keep values of an earlier tcgen05.ld behind the (preceding, volatile) wait::ld
__device__ __forceinline__ void tm_pin8(float (&v)[8]) {
  asm volatile("" : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7]));
}

template <int P, int S, int NW_ = 4>
struct SymGeom {
  static constexpr int C = 4;                 // columns per lane
  static constexpr int NW = NW_;              // warps per CTA (stacked vertically): 4, or 8 (one CTA/SM)
  static constexpr int T = 32;                // output rows per warp
  static constexpr int NT = 32 * NW;
  static constexpr int TWO = 128 - 2 * S;     // output columns per strip
  static constexpr int TH = NW * T;           // output rows per CTA
  static constexpr int SW = (128 + 2 * S + 2 * P + 3) / 4 * 4;  // smem row (floats), col j <-> X - 2S - P + j
  static constexpr int SH0 = TH + 2 * (S + P) + 1;               // smem rows used, row i <-> Y - S - P - 1 + i
  static constexpr int SH = SH0;
  static constexpr int NCW = C + 2 * P;       // centre window of a lane (H)
  static constexpr int NSW = C + 2 * P + 2 * S;  // shifted window (H, every ox)
  static constexpr int NIW = C + 2 * S;       // accumulation window u(q + o), and the partner window
  static constexpr int WARP_COLS = 8 * T;     // num[4] den[4] per row
  static constexpr int TMEM_COLS = WARP_COLS * (NW / 4);  // warps w and w+4 share a lane quadrant
  // at least 77 KB: never three CTAs on an SM (two CTAs x 256 columns fill the 512 TMEM columns; a
  // third would spin in tcgen05.alloc until one of them finishes)
  static constexpr size_t tile_bytes = (size_t)SW * SH * sizeof(float);
  static constexpr size_t smem_bytes = tile_bytes > 77 * 1024 ? tile_bytes : 77 * 1024;
  static_assert(S >= 1 && S <= 8, "partner exchange reaches two lanes");
  static_assert(WARP_COLS == 256 && (NW == 4 || NW == 8), "two 4-warp CTAs or one 8-warp CTA fill the 512 TMEM columns");
};

// N consecutive floats starting OFF floats after a 16-byte aligned lane base, via LDS.128
template <int OFF, int N>
__device__ __forceinline__ void sym_ld_win(const float* base, float (&v)[N]) {
  constexpr int A = OFF & ~3;
  constexpr int NQ = (OFF + N - A + 3) / 4;
  float tmp[4 * NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const float4 f = reinterpret_cast<const float4*>(base + A)[q];
    tmp[4 * q] = f.x; tmp[4 * q + 1] = f.y; tmp[4 * q + 2] = f.z; tmp[4 * q + 3] = f.w;
  }
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = tmp[OFF - A + i];
}

// The pairs of search row OY (1..S): S pairs (ox, ox+1) of row OY covering ox = -S..S-1, and one
// mixed pair: (S, OY) with (OY, 0) -- the S offsets of search row 0 (0 < ox <= S) ride in the
// last pair of the S passes, so no lane is idle and row 0 needs no walk of its own.
template <int P, int S, int OY>
struct SymPass {
  static constexpr int NPAIR = S + 1;
  __host__ __device__ static constexpr bool mixed(int g) { return g == S; }
  __host__ __device__ static constexpr int oxa(int g) { return mixed(g) ? S : -S + 2 * g; }
};

// true when the normal pair g, column k is the first (in the unrolled g-major order) to write the
// partner window entry k + 2g: that write assigns instead of accumulating into 0
__host__ __device__ constexpr bool sym_first_pn(int g, int k) {
  for (int gg = 0; gg < g; ++gg)
    if (k + 2 * g - 2 * gg >= 0 && k + 2 * g - 2 * gg < 4) return false;
  return true;
}

// the two lanes' differences u(q) - u(q+o) at window index t of the pair g
// (half a at window index t of column k, half b at index t - 1 of column k - 1: "b lags")
template <int P, int S, int OY, int G_>
__device__ __forceinline__ float2 sym_df(const float* c18, const float* s18, int t) {
  using Q = SymPass<P, S, OY>;
  if (Q::mixed(G_))
    return make_float2(__fsub_rn(c18[t + S], s18[t + 2 * S]), __fsub_rn(c18[t + S - 1], c18[t + OY + S - 1]));
  const float sj = s18[t + Q::oxa(G_) + S];
  return s2_sub(make_float2(c18[t + S], c18[t + S - 1]), make_float2(sj, sj));
}

template <int P, int S, int OY, int G_>
__device__ __forceinline__ void sym_df_all(const float* c18, const float* s18, float2 (&df)[4 + 2 * P]) {
#pragma unroll
  for (int t = 0; t < 4 + 2 * P; ++t) df[t] = sym_df<P, S, OY, G_>(c18, s18, t);
}

// D[g][k] += H_g(column k, image row r): the walk's initial window
template <int P, int S, int OY, int G_ = 0>
__device__ __forceinline__ void sym_acc_H_g(float2 (&D)[S + 1][4], const float* c18, const float* s18) {
  constexpr int C = 4, NCW = C + 2 * P;
  float2 df[NCW];
  sym_df_all<P, S, OY, G_>(c18, s18, df);
  float2 a = s2_mul(df[0], df[0]);
#pragma unroll
  for (int t = 1; t <= 2 * P; ++t) a = s2_fma(df[t], df[t], a);
  D[G_][0] = s2_add(D[G_][0], a);
#pragma unroll
  for (int k = 1; k < C; ++k) {
    a = s2_fma(df[k + 2 * P], df[k + 2 * P], a);
    a = s2_fma(make_float2(-df[k - 1].x, -df[k - 1].y), df[k - 1], a);
    D[G_][k] = s2_add(D[G_][k], a);
  }
  if constexpr (G_ < S) sym_acc_H_g<P, S, OY, G_ + 1>(D, c18, s18);
}

// H_g(column k) of every pair at one image row (squares chains, two distinct register pairs per
// FFMA2), into Hr[g][2k], Hr[g][2k+1] -- the layout of the TMEM ring (8 words per pair)
template <int P, int S, int OY, int G_ = 0>
__device__ __forceinline__ void sym_H_all(float (&Hr)[S + 1][8], const float* c18, const float* s18) {
  constexpr int C = 4, NCW = C + 2 * P;
  float2 df[NCW];
  sym_df_all<P, S, OY, G_>(c18, s18, df);
  float2 a = s2_mul(df[0], df[0]);
#pragma unroll
  for (int t = 1; t <= 2 * P; ++t) a = s2_fma(df[t], df[t], a);
  Hr[G_][0] = a.x;
  Hr[G_][1] = a.y;
#pragma unroll
  for (int k = 1; k < C; ++k) {
    a = s2_fma(df[k + 2 * P], df[k + 2 * P], a);
    a = s2_fma(make_float2(-df[k - 1].x, -df[k - 1].y), df[k - 1], a);
    Hr[G_][2 * k] = a.x;
    Hr[G_][2 * k + 1] = a.y;
  }
  if constexpr (G_ < S) sym_H_all<P, S, OY, G_ + 1>(Hr, c18, s18);
}

// D[g][k] += H_g(new row) - H_g(old row).  Per window index t the two squares enter as one
// product: dn^2 - dd^2 = (dn - dd)(dn + dd), and with dn = cn - sn, dd = co - so
//   dn - dd = (cn - co) - (sn - so),   dn + dd = (cn + co) - (sn + so),
// whose four row sums / differences are shared by every pair of the row (formed once per step):
// per pair and t two FADD2 and one FFMA2 link of the sliding chain instead of two FADD2 and two
// FFMA2 links.
template <int P, int S, int OY, int G_ = 0>
__device__ __forceinline__ void sym_slide_pq(float2 (&D)[S + 1][4], const float* Cd, const float* Cs,
                                             const float* Sd, const float* Ss, const float2* CdL,
                                             const float2* CsL) {
  using Q = SymPass<P, S, OY>;
  constexpr int C = 4, NCW = C + 2 * P;
  float2 pp[NCW], qq[NCW];
#pragma unroll
  for (int t = 0; t < NCW; ++t) {
    if (Q::mixed(G_)) {  // halves from two windows: scalar (b lags: column k - 1)
      pp[t] = make_float2(__fsub_rn(Cd[t + S], Sd[t + 2 * S]), __fsub_rn(Cd[t + S - 1], Cd[t + OY + S - 1]));
      qq[t] = make_float2(__fsub_rn(Cs[t + S], Ss[t + 2 * S]), __fsub_rn(Cs[t + S - 1], Cs[t + OY + S - 1]));
    } else {  // (Cd[t+S], Cd[t+S-1]) - Sd[j] broadcast
      const int j = t + Q::oxa(G_) + S;
      pp[t] = s2_sub(CdL[t], make_float2(Sd[j], Sd[j]));
      qq[t] = s2_sub(CsL[t], make_float2(Ss[j], Ss[j]));
    }
  }
  float2 a = s2_mul(pp[0], qq[0]);
#pragma unroll
  for (int t = 1; t <= 2 * P; ++t) a = s2_fma(pp[t], qq[t], a);
  D[G_][0] = s2_add(D[G_][0], a);
#pragma unroll
  for (int k = 1; k < C; ++k) {
    a = s2_fma(pp[k + 2 * P], qq[k + 2 * P], a);
    a = s2_fma(make_float2(-pp[k - 1].x, -pp[k - 1].y), qq[k - 1], a);
    D[G_][k] = s2_add(D[G_][k], a);
  }
  if constexpr (G_ < S) sym_slide_pq<P, S, OY, G_ + 1>(D, Cd, Cs, Sd, Ss, CdL, CsL);
}

template <int P, int S, int OY>
__device__ __forceinline__ void sym_slide_H(float2 (&D)[S + 1][4], const float* cn, const float* sn,
                                            const float* co, const float* so) {
  constexpr int NSW = 4 + 2 * P + 2 * S;
  static_assert(NSW % 2 == 0, "window in float2 pairs");
  float Cd[NSW], Cs[NSW], Sd[NSW], Ss[NSW];
#pragma unroll
  for (int j = 0; j < NSW; j += 2) {
    const float2 a = make_float2(cn[j], cn[j + 1]), b = make_float2(co[j], co[j + 1]);
    const float2 c = make_float2(sn[j], sn[j + 1]), d = make_float2(so[j], so[j + 1]);
    const float2 cd = s2_sub(a, b), cs = s2_add(a, b), sd = s2_sub(c, d), ss = s2_add(c, d);
    Cd[j] = cd.x; Cd[j + 1] = cd.y; Cs[j] = cs.x; Cs[j + 1] = cs.y;
    Sd[j] = sd.x; Sd[j + 1] = sd.y; Ss[j] = ss.x; Ss[j + 1] = ss.y;
  }
  // the lagged centre pairs (C[t+S], C[t+S-1]), formed once per step and shared by every pair:
  // an aligned FADD2 result read swapped where t + S is odd, two scalar operations otherwise
  constexpr int NCW = 4 + 2 * P;
  float2 CdL[NCW], CsL[NCW];
#pragma unroll
  for (int t = 0; t < NCW; ++t) {
    const int m = t + S;
    if (m & 1) {
      CdL[t] = make_float2(Cd[m], Cd[m - 1]);
      CsL[t] = make_float2(Cs[m], Cs[m - 1]);
    } else {
      CdL[t] = make_float2(__fsub_rn(cn[m], co[m]), __fsub_rn(cn[m - 1], co[m - 1]));
      CsL[t] = make_float2(__fadd_rn(cn[m], co[m]), __fadd_rn(cn[m - 1], co[m - 1]));
    }
  }
  sym_slide_pq<P, S, OY>(D, Cd, Cs, Sd, Ss, CdL, CsL);
}

// One search row OY of the warp's walk (with the mixed pair's row-0 offset).  U: smem tile;
// wrow0: smem row of the warp's d-row 0; tm: the thread's TMEM address (column 0).
template <int P, int S, int OY, bool RING>
__device__ __forceinline__ void sym_pass(const float* U, int wrow0, int lane, uint32_t tm, float2 nc) {
  using G = SymGeom<P, S>;
  using Q = SymPass<P, S, OY>;
  constexpr int C = G::C, SW = G::SW, T = G::T, NIW = G::NIW, NSW = G::NSW, NP = Q::NPAIR;
  const float* Ul = U + 4 * lane;
  auto row = [&](int y) { return Ul + (wrow0 + y) * SW; };

  float2 D[NP][C];
#pragma unroll
  for (int g = 0; g < NP; ++g)
#pragma unroll
    for (int k = 0; k < C; ++k) D[g][k] = make_float2(0.0f, 0.0f);
  constexpr int y0 = -OY;
  // d(y0) + H(y0-P-1): the first step subtracts that row again
  // RING: H of the last 2P+1 rows kept in tensor memory (columns 8T.., slot r mod (2P+1), 8 words
  // per pair), so a step computes only the row entering the window
  constexpr int NSLOT = 2 * P + 1;
  const uint32_t ring = tm + 8 * T;
#pragma unroll 1
  for (int r = y0 - P - 1; r <= y0 + P - 1; ++r) {
    float c18[NSW], s18[NSW];
    sym_ld_win<0, NSW>(row(r), c18);
    sym_ld_win<0, NSW>(row(r + OY), s18);
    if constexpr (RING) {
      float Hr[NP][8];
      sym_H_all<P, S, OY>(Hr, c18, s18);
      const int slot = (r + 64 * NSLOT) % NSLOT;
#pragma unroll
      for (int g = 0; g < NP; ++g) {
#pragma unroll
        for (int k = 0; k < C; ++k) D[g][k] = s2_add(D[g][k], make_float2(Hr[g][2 * k], Hr[g][2 * k + 1]));
        tm_st8(ring + 8 * (slot * NP + g), Hr[g]);
      }
    } else {
      sym_acc_H_g<P, S, OY>(D, c18, s18);
    }
  }
  int slot = (y0 + P + 64 * NSLOT) % NSLOT;  // slot of row y + P == slot of row y - P - 1

#pragma unroll 1
  for (int y = y0; y < T; ++y) {
    if constexpr (RING) {
      float Ho[NP][8], Hn[NP][8];
      const uint32_t sa = ring + 8 * (slot * NP);
      tm_wait_st();  // the previous step's stores (this slot was written 2P+1 steps ago)
#pragma unroll
      for (int g = 0; g < NP; ++g) tm_ld8(sa + 8 * g, Ho[g]);
      float cn[NSW], sn[NSW];
      sym_ld_win<0, NSW>(row(y + P), cn);
      sym_ld_win<0, NSW>(row(y + P + OY), sn);
      sym_H_all<P, S, OY>(Hn, cn, sn);
      tm_wait_ld();
#pragma unroll
      for (int g = 0; g < NP; ++g) tm_pin8(Ho[g]);
#pragma unroll
      for (int g = 0; g < NP; ++g) {
#pragma unroll
        for (int k = 0; k < C; ++k)
          D[g][k] = s2_add(D[g][k], s2_sub(make_float2(Hn[g][2 * k], Hn[g][2 * k + 1]),
                                           make_float2(Ho[g][2 * k], Ho[g][2 * k + 1])));
        tm_st8(sa + 8 * g, Hn[g]);
      }
      slot = slot + 1 == NSLOT ? 0 : slot + 1;
    } else {
      float cn[NSW], sn[NSW], co[NSW], so[NSW];
      sym_ld_win<0, NSW>(row(y + P), cn);
      sym_ld_win<0, NSW>(row(y + P + OY), sn);
      sym_ld_win<0, NSW>(row(y - P - 1), co);
      sym_ld_win<0, NSW>(row(y - P - 1 + OY), so);
      sym_slide_H<P, S, OY>(D, cn, sn, co, so);
    }
    float ia[NIW], iy[NIW];
    sym_ld_win<P, NIW>(row(y + OY), ia);  // u(q + o): window index m + S, m = column - (X - S + 4 lane)
    sym_ld_win<P, NIW>(row(y), iy);       // row y: u(q) = iy[k + S], and u(q + (OY, 0))
    float2 A[C], B[C], Pn[NIW], Pd[NIW];
    float Zn[C], Zd[C];  // the mixed pair's row-0 partner contributions, by source column
#pragma unroll
    for (int k = 0; k < C; ++k) {
      A[k] = B[k] = make_float2(0.0f, 0.0f);
      Zn[k] = Zd[k] = 0.0f;
    }
#pragma unroll
    for (int j = 0; j < NIW; ++j) Pn[j] = Pd[j] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int g = 0; g < NP; ++g)
#pragma unroll
      for (int k = 0; k < C; ++k) {
        // sliding sums can round below 0; a negative d with a tiny h would give w = inf (R29)
        const float2 t = s2_mul(make_float2(fmaxf(D[g][k].x, 0.0f), fmaxf(D[g][k].y, 0.0f)), nc);
        const float2 w = make_float2(ex2_approx(t.x), ex2_approx(t.y));
        const float uq = iy[k + S], uqb = iy[k + S - 1];  // u(q) of half a (column k), half b (k - 1)
        const bool first = g == 0;  // first write of A[k], B[k] (resolved at compile time)
        B[k] = first ? w : s2_add(B[k], w);
        if (Q::mixed(g)) {
          A[k].x = fmaf(w.x, ia[k + 2 * S], A[k].x);
          A[k].y = fmaf(w.y, iy[k + OY + S - 1], A[k].y);
          if (k < 2) {  // entries 2S, 2S + 1 were written by the last normal pair
            Pn[k + 2 * S].x = fmaf(w.x, uq, Pn[k + 2 * S].x);  // partner (q + (S, OY)): row y + OY
            Pd[k + 2 * S].x += w.x;
          } else {
            Pn[k + 2 * S].x = w.x * uq;
            Pd[k + 2 * S].x = w.x;
          }
          Zn[k] = w.y * uqb;  // partner (q + (OY, 0)) of source column k - 1: row y, column k - 1 + OY
          Zd[k] = w.y;
        } else {
          const int ja = k + Q::oxa(g) + S;  // window index of column k + oxa (both halves)
          const float2 qa = make_float2(ia[ja], ia[ja]);
          A[k] = first ? s2_mul(w, qa) : s2_fma(w, qa, A[k]);
          if (sym_first_pn(g, k)) {
            Pn[ja] = s2_mul(w, make_float2(uq, uqb));  // both halves -> column ja
            Pd[ja] = w;
          } else {
            Pn[ja] = s2_fma(w, make_float2(uq, uqb), Pn[ja]);
            Pd[ja] = s2_add(Pd[ja], w);
          }
        }
      }
    // partner window of row y + OY: column J collects Pn[J].x and Pn[J].y; columns outside
    // [S, S+C) belong to the lanes 1..2 to the left / right
    float on[NIW], od[NIW];
#pragma unroll
    for (int j = 0; j < NIW; ++j) {
      on[j] = Pn[j].x + Pn[j].y;
      od[j] = Pd[j].x + Pd[j].y;
    }
    float rn[C], rd[C], zn[C], zd[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      rn[k] = on[k + S];
      rd[k] = od[k + S];
      zn[k] = k + 1 >= OY ? Zn[k + 1 - OY] : 0.0f;  // source column k + 1 - OY - 1
      zd[k] = k + 1 >= OY ? Zd[k + 1 - OY] : 0.0f;
    }
#pragma unroll
    for (int dl = 1; dl <= 2; ++dl)
#pragma unroll
      for (int k = 0; k < C; ++k) {
        // from lane - dl: its window index k + 4 dl + S
        if (k + 4 * dl + S < NIW) {
          rn[k] += __shfl_up_sync(0xffffffffu, on[k + 4 * dl + S], dl);
          rd[k] += __shfl_up_sync(0xffffffffu, od[k + 4 * dl + S], dl);
        }
        // from lane + dl: its window index k - 4 dl + S
        if (k - 4 * dl + S >= 0) {
          rn[k] += __shfl_down_sync(0xffffffffu, on[k - 4 * dl + S], dl);
          rd[k] += __shfl_down_sync(0xffffffffu, od[k - 4 * dl + S], dl);
        }
        // row-0 partner: entry k + 4 dl + 1 - OY of lane - dl (its source column one less)
        if (k + 4 * dl + 1 - OY >= 0 && k + 4 * dl + 1 - OY < C) {
          zn[k] += __shfl_up_sync(0xffffffffu, Zn[k + 4 * dl + 1 - OY], dl);
          zd[k] += __shfl_up_sync(0xffffffffu, Zd[k + 4 * dl + 1 - OY], dl);
        }
      }
    // TMEM read-modify-write: own row y (own pairs + the row-0 partners), partner row y + OY
    const bool own_ok = y >= 0;
    const bool par_ok = y + OY < T;
    float vo[8], vp[8];
    tm_wait_st();
    if (own_ok) tm_ld8(tm + 8 * y, vo);
    if (par_ok) tm_ld8(tm + 8 * (y + OY), vp);
    tm_wait_ld();
    if (own_ok) tm_pin8(vo);
    if (par_ok) tm_pin8(vp);
    // own sums: column k = half a of k + half b of k + 1 (k = 3: lane + 1's column 0; lane 31's
    // column 3 and lane 0's column -1 are halo columns, never output)
    const float an = __shfl_down_sync(0xffffffffu, A[0].y, 1), bd = __shfl_down_sync(0xffffffffu, B[0].y, 1);
    if (own_ok) {
#pragma unroll
      for (int k = 0; k < C; ++k) {
        vo[k] += (A[k].x + (k + 1 < C ? A[k + 1].y : an)) + zn[k];
        vo[4 + k] += (B[k].x + (k + 1 < C ? B[k + 1].y : bd)) + zd[k];
      }
      tm_st8(tm + 8 * y, vo);
    }
    if (par_ok) {
#pragma unroll
      for (int k = 0; k < C; ++k) {
        vp[k] += rn[k];
        vp[4 + k] += rd[k];
      }
      tm_st8(tm + 8 * (y + OY), vp);
    }
  }
}

template <int P, int S, bool RING, int OY = 1>
__device__ __forceinline__ void sym_passes(const float* U, int wrow0, int lane, uint32_t tm, float2 nc) {
  sym_pass<P, S, OY, RING>(U, wrow0, lane, tm, nc);
  // keep the CTA's warps in the same pass: they then share the instruction fetch of one pass body
  // (~0.4% faster; a barrier every step or every 4 steps costs 3%)
  __syncthreads();
  if constexpr (OY < S) sym_passes<P, S, RING, OY + 1>(U, wrow0, lane, tm, nc);
}

// RING = false: 2 CTAs/SM, 256 TMEM columns each (num/den), the slide recomputes the leaving row.
// RING = true ("sym_ring"): 1 CTA/SM with all 512 columns: num/den + the H ring of the last 2P+1 rows.
// NW = 8 ("sym_tmem8"): one 8-warp CTA per SM (256 x 118 tiles); its warps run each pass together.
template <int P, int S, bool RING, int NW = 4>
__global__ void __launch_bounds__(32 * NW, (RING || NW == 8) ? 1 : 2) nlm_sym(NlmParams p, int ntx, int nty,
                                                                              int use_async) {
  using G = SymGeom<P, S, NW>;
  constexpr int TMEM_COLS = RING ? 512 : G::TMEM_COLS;
  static_assert(!RING || (NW == 4 && G::WARP_COLS + 8 * (2 * P + 1) * (S + 1) <= 512), "ring fits the tensor memory");
  constexpr int C = G::C, SW = G::SW, SH = G::SH, T = G::T, TWO = G::TWO, TH = G::TH;
  extern __shared__ __align__(128) float U[];
  __shared__ uint32_t tm_base_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const int per_img = ntx * nty;
  const int b = blockIdx.x / per_img;
  const int rr = blockIdx.x - b * per_img;
  const int X = (rr % ntx) * TWO;  // first output column
  const int Y = (rr / ntx) * TH;   // first output row (local)
  const int gY = p.dst.y0 + Y;
  const int c0 = X - 2 * S - P, r0 = gY - S - P - 1;  // image column / global row of smem (0, 0)
  // interior tiles (no boundary inside the tile) take the asynchronous copy
  const bool async_tile = use_async && (c0 & 1) == 0 && c0 >= 0 && c0 + SW <= p.src.W && r0 >= 0 && r0 + G::SH0 <= p.src.Hg;

  if (warp == 0) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&tm_base_sh);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst), "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (async_tile) {
    // interior tile: 8-byte cp.async (LDGSTS.64) of every row, all in flight at once; rows past
    // the band buffer are zero (read_B returns 0 there)
    constexpr int HW = SW / 2;  // float2 per row
#pragma unroll 4
    for (int i = tid; i < HW * SH; i += G::NT) {
      const int r = i / HW, c = i - r * HW;
      const int lr = r0 + r - p.src.y0;
      float2* dst = reinterpret_cast<float2*>(U + r * SW) + c;
      if ((unsigned)lr < (unsigned)p.src.Hl) {
        const float* src = reinterpret_cast<const float*>(p.src.base + (int64_t)b * p.src.bstride + (int64_t)lr * p.src.pitch) + c0 + 2 * c;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
      } else {
        *dst = make_float2(0.0f, 0.0f);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
    // image tile, boundary applied at load time (8 loads in flight per thread)
    constexpr int N = SW * SH, STEP = G::NT * 8;
#pragma unroll 1
    for (int i0 = 0; i0 < N; i0 += STEP) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * G::NT + tid;
        const int r = i / SW, c = i - r * SW;
        v[u] = i < N ? read_B(p.src, b, c0 + c, r0 + r) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * G::NT + tid;
        if (i < N) U[i] = v[u];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tm_base_sh + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(G::WARP_COLS * (warp >> 2));
  const int wrow0 = warp * T + S + P + 1;  // smem row of the warp's output row 0
  const float* Ul = U + 4 * lane;

  // centre pair: num = u(p), den = 1
#pragma unroll 1
  for (int y = 0; y < T; ++y) {
    float io[C];
    sym_ld_win<S + P, C>(Ul + (wrow0 + y) * SW, io);
    float v[8] = {io[0], io[1], io[2], io[3], 1.0f, 1.0f, 1.0f, 1.0f};
    tm_st8(tm + 8 * y, v);
  }
  const float2 nc = make_float2(-p.coef, -p.coef);
  sym_passes<P, S, RING>(U, wrow0, lane, tm, nc);

  tm_wait_st();
  const int x0 = X - S + 4 * lane;
#pragma unroll 1
  for (int y = 0; y < T; ++y) {
    float v[8];
    tm_ld8(tm + 8 * y, v);
    tm_wait_ld();
    tm_pin8(v);
    const int ly = Y + warp * T + y;
    if (ly < p.dst.H) {
      float* drow = dst_row(p.dst, b, ly);
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const int x = x0 + k;
        if (x >= X && x < X + TWO && x < p.src.W) drow[x] = __fdiv_rn(v[k], v[4 + k]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base_sh), "n"(TMEM_COLS));
  }
}

template <int P, int S, bool RING = false, int NW = 4>
inline cudaError_t launch_sym(const NlmParams& p, int batch, cudaStream_t s) {
  using G = SymGeom<P, S, NW>;
  static_assert(NW == 8 || G::smem_bytes <= 113 * 1024, "two CTAs per SM");
  static_assert(G::smem_bytes <= 227 * 1024, "shared memory");
  auto kern = nlm_sym<P, S, RING, NW>;
  // RING / NW = 8 hold all 512 TMEM columns: shared memory above half the SM's so a second CTA never
  // waits in tcgen05.alloc
  const bool one = RING || NW == 8;
  const size_t smem = one ? (G::smem_bytes > 115 * 1024 ? G::smem_bytes : 115 * 1024) : G::smem_bytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int ntx = (p.src.W + G::TWO - 1) / G::TWO, nty = (p.dst.H + G::TH - 1) / G::TH;
  const long long nblk = (long long)ntx * nty * batch;
  if (nblk <= 0) return cudaSuccess;
  if (nblk > 0x7fffffffLL) return cudaErrorInvalidValue;
  // the asynchronous tile copy moves 8-byte pairs: base, pitch and image stride 8-byte aligned
  const int use_async = ((uintptr_t)p.src.base % 8 == 0) && (p.src.pitch % 8 == 0) && (batch == 1 || p.src.bstride % 8 == 0);
  kern<<<(unsigned)nblk, G::NT, smem, s>>>(p, ntx, nty, use_async);
  count_launch();
  return cudaGetLastError();
}

}  // namespace icl
