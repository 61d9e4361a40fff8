// Retired (DESIGN.md §5 "Tried and retired"): row-reuse Harris interior path.
// 8 x 4096^2: 0.527 ms vs 0.423 ms for harris_shfl_interior -- the unrolled
// 5-step body (needed for a static carry rotation) hits the 128-register cap
// and the instruction cache; kept for reference, not built.
// Row-reuse form of harris_shfl_interior ("shfl_*_rr" variants): a step needs
// the three input rows u, u+1, u+2, of which two were already read by the
// previous step -- so each step loads ONE new smem row (1 LDS.128 + 2 SHFL
// instead of 3 + 6) and computes the horizontal differences hd of that row
// only, carrying (row, hd) of the two previous rows in registers (the step
// loop of a block is unrolled so the carry rotates statically).  Sxy's
// vertical running sums are packed in float2 lanes per output pair.  The
// per-output fp32 operations are exactly those of harris_shfl_interior
// (bit-identical).
template <int B, int NW>
__device__ __forceinline__ void harris_shfl_interior_rr(const HarrisParams& p, int S, float* smem) {
  constexpr int A = B / 2;
  constexpr int BB = B - 1 - A;
  constexpr int NT = 32 * NW;
  constexpr int HP = 8;
  constexpr int TW = 120 * NW;
  constexpr int ROWLEN = TW + 2 * HP;
  constexpr int NSLOT = ROWLEN / 4;
  constexpr int RB = HarFastGeom<B>::RB, NBLKS = HarFastGeom<B>::NBLKS, NSR = HarFastGeom<B>::NSR;
  static_assert(RB >= 2, "mirror rows cover the two rows a step reads past its block");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TW;
  const int ly0 = blockIdx.y * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  const int NY = (ly1 - ly0) + B - 1;
  const int NL = NY + 2;
  const int NBI = (NY + RB - 1) / RB;
  const int NBL = (NL + RB - 1) / RB;
  const int64_t spitch = p.src.pitch >> 2;
  const bool loader = tid < NSLOT;
  const float* gsrc = src_row(p.src, b, g0 - A - 1) + (x0 - HP + 4 * tid);
  float* sdst = smem + 4 * tid;

  auto load_block = [&](int m) {
    if (!loader) return;
    const float* g = gsrc + (int64_t)(m * RB) * spitch;
    const int r0 = (m % NBLKS) * RB;
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      if (m * RB + u < NL) {
        cp_async16(sdst + (r0 + u) * ROWLEN, g, 16);
        if (u < 2 && r0 == 0) cp_async16(sdst + (NSR + u) * ROWLEN, g, 16);  // mirror
      }
      g += spitch;
    }
  };
  for (int m = 0; m < NBLKS - 1; ++m) {
    if (m < NBL) load_block(m);
    cp_async_commit();
  }

  const int xl = x0 + 120 * warp + 4 * (lane - 1);
  const float* stb = smem + (xl - (x0 - HP));
  const bool emit = lane >= 1 && lane <= 30;
  constexpr int NC = B > 1 ? B - 1 : 1;
  float2 c2[NC][4];
  float2 cxy[NC][2];  // (output q = 2m, 2m+1)
#pragma unroll
  for (int k = 0; k < NC; ++k) {
#pragma unroll
    for (int q = 0; q < 4; ++q) c2[k][q] = make_float2(0.0f, 0.0f);
    cxy[k][0] = cxy[k][1] = make_float2(0.0f, 0.0f);
  }
  float* drow = dst_row(p.dst, b, ly0) + xl;
  const int64_t dpitch = p.dst.pitch >> 2;
  char* mrow = p.mask ? p.mask + (int64_t)b * p.mbstride + (int64_t)ly0 * p.mpitch + xl : nullptr;

  // one smem row -> columns xl-1 .. xl+4 (index c+1 <-> column xl+c) and hd(c) = in(c+2) - in(c)
  auto fetch = [&](const float* sr, float (&in)[6], float (&hd)[4]) {
    const float4 w = *reinterpret_cast<const float4*>(sr);
    in[0] = __shfl_up_sync(0xffffffffu, w.w, 1);
    in[1] = w.x; in[2] = w.y; in[3] = w.z; in[4] = w.w;
    in[5] = __shfl_down_sync(0xffffffffu, w.x, 1);
#pragma unroll
    for (int c = 0; c < 4; ++c) hd[c] = __fsub_rn(in[c + 2], in[c]);
  };
  float in0[6], in1[6], hd0[4], hd1[4];  // carried rows (step's rows 0 and 1)

#pragma unroll 1
  for (int i = 0; i < NBI; ++i) {
    cp_async_wait<NBLKS - 3>();
    __syncthreads();
    if (i + NBLKS - 1 < NBL) load_block(i + NBLKS - 1);
    cp_async_commit();
    const float* sb = stb + (i % NBLKS) * RB * ROWLEN;
    if (i == 0) {
      fetch(sb, in0, hd0);
      fetch(sb + ROWLEN, in1, hd1);
    }
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int step = i * RB + u;
      if (step < NY) {
        float in2[6], hd2[4];
        fetch(sb + (u + 2) * ROWLEN, in2, hd2);
        float vd[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) vd[c] = __fsub_rn(in2[c], in0[c]);
        float2 g[8];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          g[c + 2].x = __fmaf_rn(2.0f, hd1[c], __fadd_rn(hd0[c], hd2[c]));
          g[c + 2].y = __fmaf_rn(2.0f, vd[c + 1], __fadd_rn(vd[c], vd[c + 2]));
        }
        g[0].x = __shfl_up_sync(0xffffffffu, g[4].x, 1);
        g[0].y = __shfl_up_sync(0xffffffffu, g[4].y, 1);
        g[1].x = __shfl_up_sync(0xffffffffu, g[5].x, 1);
        g[1].y = __shfl_up_sync(0xffffffffu, g[5].y, 1);
        g[6].x = __shfl_down_sync(0xffffffffu, g[2].x, 1);
        g[6].y = __shfl_down_sync(0xffffffffu, g[2].y, 1);
        g[7].x = __shfl_down_sync(0xffffffffu, g[3].x, 1);
        g[7].y = __shfl_down_sync(0xffffffffu, g[3].y, 1);
        float2 h2[4];
        float2 hxy[2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 hxxyy = make_float2(0.0f, 0.0f);
          float hh = 0.0f;
#pragma unroll
          for (int t = -A; t <= BB; ++t) {
            const float2 gg = g[2 + q + t];
            hxxyy = __ffma2_rn(gg, gg, hxxyy);
            hh = __fmaf_rn(gg.x, gg.y, hh);
          }
          h2[q] = hxxyy;
          if (q & 1) hxy[q >> 1].y = hh; else hxy[q >> 1].x = hh;
        }
        float2 s2o[4];
        float2 sxyo[2];
        if (B > 1) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            s2o[q] = __fadd2_rn(c2[0][q], h2[q]);  // completes output row step-B+1
#pragma unroll
            for (int k = 0; k + 1 < NC; ++k) c2[k][q] = __fadd2_rn(c2[k + 1][q], h2[q]);
            c2[NC - 1][q] = h2[q];
          }
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            sxyo[m] = __fadd2_rn(cxy[0][m], hxy[m]);
#pragma unroll
            for (int k = 0; k + 1 < NC; ++k) cxy[k][m] = __fadd2_rn(cxy[k + 1][m], hxy[m]);
            cxy[NC - 1][m] = hxy[m];
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) s2o[q] = h2[q];
          sxyo[0] = hxy[0];
          sxyo[1] = hxy[1];
        }
        if (step >= B - 1) {
          float R[4];
          R[0] = harris_R(s2o[0].x, sxyo[0].x, s2o[0].y, p.k);
          R[1] = harris_R(s2o[1].x, sxyo[0].y, s2o[1].y, p.k);
          R[2] = harris_R(s2o[2].x, sxyo[1].x, s2o[2].y, p.k);
          R[3] = harris_R(s2o[3].x, sxyo[1].y, s2o[3].y, p.k);
          if (emit) {
            st_cs4(drow, make_float4(R[0], R[1], R[2], R[3]));
            if (mrow)
              *reinterpret_cast<uchar4*>(mrow) =
                  make_uchar4(R[0] > p.threshold, R[1] > p.threshold, R[2] > p.threshold, R[3] > p.threshold);
          }
          drow += dpitch;
          if (mrow) mrow += p.mpitch;
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) { in0[c] = in1[c]; in1[c] = in2[c]; }
#pragma unroll
        for (int c = 0; c < 4; ++c) { hd0[c] = hd1[c]; hd1[c] = hd2[c]; }
      }
    }
  }
  cp_async_wait<0>();
}

