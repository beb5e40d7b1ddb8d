// Device arithmetic of the Van Oosterom-Strackee (VOS) solid angle for the
// B200 labeling kernels. SPEC.md:225-233, 261 (per-triangle closed form):
//   Omega/2 = atan2(num, den),  num = R1.(R2 x R3),
//   den = r1 r2 r3 + (R1.R2) r3 + (R1.R3) r2 + (R2.R3) r1,  R_i = v_i - p.
//
// fp32 pass. num is evaluated as N.R1 with N = (v2-v1) x (v3-v1) precomputed
// in fp64 per triangle (det[R1,R2,R3] = det[R1, v2-v1, v3-v1]); this is the
// same quantity as the cross/dot form with ~1e4x less cancellation for far
// points, and 6 fewer FP32 ops. Every operation is an explicit _rn intrinsic:
// no contraction or reassociation is left to the compiler. Which evaluator
// (far or near, below) a (point, 8-triangle group) pair uses depends only on
// that point's own distance test, so a point's s never depends on its warp
// mates, hence not on sharding or ordering.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

namespace nm {

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Far-range arctangent in the near evaluator: atan(x) = x (1 + c1 y + c2 y^2
// + c3 y^3), y = x^2, used for |x| <= kFarX (truncation x^9/9 < 2e-9
// relative, far below fp32 rounding); full-range atan2_near otherwise.
constexpr float kFarX = 0.125f;

// ---------------------------------------------------------------------------
// Packed form: two points per float2 lane pair, triangle operands broadcast.
// sm_100a executes FADD2/FMUL2/FFMA2 (fp32x2) with a scalar register
// broadcast to both lanes (".F32" operand), halving the FP32 issue slots per
// evaluation. Every lane op is an IEEE fp32 _rn operation, bit-identical to
// the scalar intrinsics above.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 bc(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

struct VosTerms2 {
  float2 num, den, r1, r2, r3;
};

// (mx, my, mz) = -(p - c) for two points.
__device__ __forceinline__ VosTerms2 vos_terms2(const float4& A, const float4& B, const float4& C, float2 mx,
                                                float2 my, float2 mz) {
  const float2 x1 = add2(bc(A.x), mx), y1 = add2(bc(A.y), my), z1 = add2(bc(A.z), mz);
  const float2 x2 = add2(bc(B.x), mx), y2 = add2(bc(B.y), my), z2 = add2(bc(B.z), mz);
  const float2 x3 = add2(bc(C.x), mx), y3 = add2(bc(C.y), my), z3 = add2(bc(C.z), mz);
  const float2 q1 = fma2(z1, z1, fma2(y1, y1, mul2(x1, x1)));
  const float2 q2 = fma2(z2, z2, fma2(y2, y2, mul2(x2, x2)));
  const float2 q3 = fma2(z3, z3, fma2(y3, y3, mul2(x3, x3)));
  VosTerms2 t;
  t.r1 = make_float2(sqrt_approx(q1.x), sqrt_approx(q1.y));
  t.r2 = make_float2(sqrt_approx(q2.x), sqrt_approx(q2.y));
  t.r3 = make_float2(sqrt_approx(q3.x), sqrt_approx(q3.y));
  t.num = fma2(bc(C.w), z1, fma2(bc(B.w), y1, mul2(bc(A.w), x1)));
  const float2 d12 = fma2(z1, z2, fma2(y1, y2, mul2(x1, x2)));
  const float2 d13 = fma2(z1, z3, fma2(y1, y3, mul2(x1, x3)));
  const float2 d23 = fma2(z2, z3, fma2(y2, y3, mul2(x2, x3)));
  t.den = fma2(fma2(t.r1, t.r2, d12), t.r3, fma2(d13, t.r2, mul2(d23, t.r1)));
  return t;
}

// The same terms in the exact double-single frame (near path of the
// triangle layout): R = (v - c) + m + l.
__device__ __forceinline__ VosTerms2 vos_terms2x(const float4& A, const float4& B, const float4& C, const float2 (&m)[3],
                                                 const float2 (&l)[3]) {
  const float2 x1 = add2(add2(bc(A.x), m[0]), l[0]), y1 = add2(add2(bc(A.y), m[1]), l[1]),
               z1 = add2(add2(bc(A.z), m[2]), l[2]);
  const float2 x2 = add2(add2(bc(B.x), m[0]), l[0]), y2 = add2(add2(bc(B.y), m[1]), l[1]),
               z2 = add2(add2(bc(B.z), m[2]), l[2]);
  const float2 x3 = add2(add2(bc(C.x), m[0]), l[0]), y3 = add2(add2(bc(C.y), m[1]), l[1]),
               z3 = add2(add2(bc(C.z), m[2]), l[2]);
  const float2 q1 = fma2(z1, z1, fma2(y1, y1, mul2(x1, x1)));
  const float2 q2 = fma2(z2, z2, fma2(y2, y2, mul2(x2, x2)));
  const float2 q3 = fma2(z3, z3, fma2(y3, y3, mul2(x3, x3)));
  VosTerms2 t;
  t.r1 = make_float2(sqrt_approx(q1.x), sqrt_approx(q1.y));
  t.r2 = make_float2(sqrt_approx(q2.x), sqrt_approx(q2.y));
  t.r3 = make_float2(sqrt_approx(q3.x), sqrt_approx(q3.y));
  t.num = fma2(bc(C.w), z1, fma2(bc(B.w), y1, mul2(bc(A.w), x1)));
  const float2 d12 = fma2(z1, z2, fma2(y1, y2, mul2(x1, x2)));
  const float2 d13 = fma2(z1, z3, fma2(y1, y3, mul2(x1, x3)));
  const float2 d23 = fma2(z2, z3, fma2(y2, y3, mul2(x2, x3)));
  t.den = fma2(fma2(t.r1, t.r2, d12), t.r3, fma2(d13, t.r2, mul2(d23, t.r1)));
  return t;
}

__device__ __forceinline__ float2 acc_far2(float2 acc, float2 num, float2 den) {
  const float2 x = mul2(num, make_float2(rcp_approx(den.x), rcp_approx(den.y)));
  const float2 y = mul2(x, x);
  const float2 p = fma2(fma2(fma2(bc(-0.142857142857f), y, bc(0.2f)), y, bc(-0.333333333333f)), y, bc(1.0f));
  return fma2(x, p, acc);
}

// Full-range atan2 for the near path: one MUFU.RCP, an odd degree-17
// near-minimax polynomial on [0,1] (|err| <= 6e-9 in exact arithmetic,
// ~1.2e-7 evaluated in fp32) and a branch-free octant fix-up. atan2(+-0, x<0)
// = +-pi and atan2(0, 0) = 0 as in C.
__device__ __forceinline__ float atan2_near(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float t = mx > 0.0f ? __fmul_rn(mn, rcp_approx(mx)) : 0.0f;
  const float s = __fmul_rn(t, t);
  float p = 0.0024567244108766317f;
  p = __fmaf_rn(p, s, -0.014401360414922237f);
  p = __fmaf_rn(p, s, 0.03978123515844345f);
  p = __fmaf_rn(p, s, -0.07234859466552734f);
  p = __fmaf_rn(p, s, 0.10498947650194168f);
  p = __fmaf_rn(p, s, -0.14161230623722076f);
  p = __fmaf_rn(p, s, 0.19985906779766083f);
  p = __fmaf_rn(p, s, -0.33332598209381104f);
  p = __fmaf_rn(p, s, 0.9999998807907104f);
  float a = __fmul_rn(t, p);
  a = ay > ax ? __fsub_rn(1.57079632679489662f, a) : a;
  a = x < 0.0f ? __fsub_rn(3.14159265358979324f, a) : a;
  return copysignf(a, y);
}

// Near path for one lane, given the packed far-range value of that lane.
__device__ __forceinline__ float acc_near_lane(float acc, float a_far, float num, float den, float r1, float r2,
                                               float r3, float tau, float delta, bool& det) {
  const bool far_range = (den > 0.0f) && (fabsf(num) <= __fmul_rn(kFarX, den));
  const float a_full = __fadd_rn(acc, atan2_near(num, den));
  const float prod = __fmul_rn(__fmul_rn(r1, r2), r3);
  const float lim = __fmul_rn(tau, prod);
  det |= ((fabsf(num) <= lim) && (den <= lim)) || (fminf(r1, fminf(r2, r3)) <= delta);
  return far_range ? a_far : a_full;
}

// ---------------------------------------------------------------------------
// Strip segments: 8 triangles t_k = (u_k, u_{k+1}, u_{k+2})
// of one triangle strip share vertices and edges, so per triangle only one
// new vertex and two new edges enter. Record (kSegF4 float4):
//   rec[0..9]   V_i  = (2x, 2y, 2z, |V_i|^2)             vertices (doubled), subtile frame
//   rec[10..17] T_k  = 2 (N_k.x, N_k.y, N_k.z, N_k.V_k)  N_k = (v2-v1)x(v3-v1) of the
//                                                        original triangle, so num_k
//                                                        carries the outward orientation
//                                                        whatever the strip's winding parity
//   rec[18..23] C_k  = -(alpha_k, beta_k, gamma_k)       the vertex dot products of
//                                                        triangle k (a, b, c = u_k,
//                                                        u_{k+1}, u_{k+2}): alpha =
//                                                        (a-c).(b-c), beta = (b-a).(c-a),
//                                                        gamma = (a-b).(c-b)
// The factor 2 on T is an exact power-of-two scaling: the far evaluator
// works with (2 num, 2 den), the near one scales back exactly.
//
// Two evaluators share the record:
//   far  (a point at >= 4 rho + 0.05 mm from the centre of the group's
//        bounding ball of radius rho):
//        q = |V|^2 + |p|^2 - 2 V.p  (4 ops, no R vector), num = N.V - N.p,
//        2 den = u v w - alpha u - beta v - gamma w  (u = r_a + r_b, v = r_b + r_c,
//                w = r_a + r_c) = w (u v - gamma) - alpha u - beta v,
//        per triangle |Omega/2| <= pi (1 - sqrt(1 - 1/16)) = 0.1004 rad there
//        (spherical-cap bound), so a consecutive pair's half-angle sum stays
//        <= 0.2 rad, where a 3-coefficient minimax odd polynomial (after the
//        complex product below) is within 4.9e-8 rad: 18.6 FP32 lane-ops +
//        1.75 MUFU;
//   near R-based terms in the exact double-single subtile frame, direct dot
//        products, 3-term series for |x| <= 0.125 else full-range atan2,
//        plus the near-surface detector.
// Which evaluator a (point, group) pair uses depends only on that point's own
// distance test, never on its warp mates (mixed warps run both and select per
// lane), so results are independent of sharding and point order.
// ---------------------------------------------------------------------------
#ifndef NM_SEG_TRIS
#define NM_SEG_TRIS 8
#endif
constexpr int kSegTris = NM_SEG_TRIS;               // triangles per segment
constexpr int kSegT = kSegTris + 2;                 // first T_k (after the vertices)
constexpr int kSegC = kSegT + kSegTris;             // first vertex-dot coefficient float4
constexpr int kSegF4 = kSegC + (3 * kSegTris + 3) / 4;  // 24 float4 for 8 triangles
constexpr float kRecScale = 2.0f;  // T_k scaling of the record (host packing)

__device__ __forceinline__ float f4_at(const float4& v, int c) {
  return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}
// -(vertex dot) coefficient i of the segment (3 per triangle), shared memory
__device__ __forceinline__ float coef_val(const float4* rec, int idx) { return f4_at(rec[kSegC + (idx >> 2)], idx & 3); }

// Per point pair, in the subtile frame: m = -(p - c); sp = |p - c|^2 (the
// subtile far test's squared distance, reused).
struct PairFrame {
  float2 mx, my, mz, sp;
};


// ---- far evaluator --------------------------------------------------------
// |V - p| from |V - p|^2 = |V|^2 + |p|^2 + (2V).(-p): 4 ops + MUFU.SQRT
__device__ __forceinline__ float2 far_dist(const float4& V, const PairFrame& f) {
  const float2 q = fma2(bc(V.x), f.mx, fma2(bc(V.y), f.my, fma2(bc(V.z), f.mz, add2(bc(V.w), f.sp))));
  return make_float2(sqrt_approx(q.x), sqrt_approx(q.y));
}

// atan(N/D) for |N/D| <= tan(0.2): x (1 + c1 x^2 + c2 x^4), minimax on
// [0, tan 0.2] with the linear term pinned to 1 (exact for small x): max
// error 4.9e-8 rad (6.2e-8 evaluated in fp32), below the 4-term Taylor
// series' 6.2e-8 (7.4e-8) at one FMA less.
__device__ __forceinline__ float2 atan_far3(float2 acc, float2 num, float2 den) {
  const float2 x = mul2(num, make_float2(rcp_approx(den.x), rcp_approx(den.y)));
  const float2 y = mul2(x, x);
  const float2 p = fma2(fma2(bc(0.1915847659111023f), y, bc(-0.3332153856754303f)), y, bc(1.0f));
  return fma2(x, p, acc);
}

// Far evaluator.
// Denominator: with 2 R_a.R_b = r_a^2 + r_b^2 - |e_ab|^2 the VOS denominator
// 2 den = 2 r_a r_b r_c + 2 (R_a.R_b r_c + R_a.R_c r_b + R_b.R_c r_a)
// regroups through (r_a + r_b)(r_b + r_c)(r_c + r_a) = sum_sym r_a^2 r_b +
// 2 r_a r_b r_c into u v w - |e_ab|^2 r_c - |e_ac|^2 r_b - |e_bc|^2 r_a, and
// substituting r_c = (v + w - u)/2 etc. into the edge terms gives
// u v w - alpha u - beta v - gamma w with the triangle's vertex dot products
// (host constants). Far away r ~ d >> |e|, so u v w (~8 d^3) dominates without
// cancellation: v, w, fma(u, v, -gamma), the alpha/beta terms (2, broadcast
// operands) and one fma = 6 ops per triangle, u carried from the previous one.
// Angle: consecutive triangles are combined pairwise through the complex
// product (den0 + i num0)(den1 + i num1), whose argument is the sum of the two
// half-angles (each <= 0.1004 rad far away, so the sum stays in the minimax
// polynomial's range and the real part stays > 0): half the MUFU.RCP of two
// separate arctangents.
// Chain state (ra, rb, sab): the distances of the segment's first two
// vertices and their sum. cont: this segment continues the previous one of
// the same strip in the same subtile, whose final state is already there.
template <int NP>
__device__ __forceinline__ void seg_far(const float4* __restrict__ rec, const PairFrame (&f)[NP], float2 (&acc)[NP],
                                        float2 (&ra)[NP], float2 (&rb)[NP], float2 (&sab)[NP], bool cont) {
  if (!cont) {
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      ra[q] = far_dist(rec[0], f[q]);
      rb[q] = far_dist(rec[1], f[q]);
      sab[q] = add2(ra[q], rb[q]);
    }
  }
  float2 n0[NP], d0[NP];
#pragma unroll
  for (int k = 0; k < kSegTris; ++k) {
    const float4 V2 = rec[k + 2];
    const float4 T = rec[kSegT + k];
    const float ca = coef_val(rec, 3 * k), cb = coef_val(rec, 3 * k + 1), cg = coef_val(rec, 3 * k + 2);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const float2 rc = far_dist(V2, f[q]);
      const float2 sbc = add2(rb[q], rc);  // v
      const float2 sac = add2(ra[q], rc);  // w
      const float2 x = fma2(sab[q], sbc, bc(cg));  // u v - gamma
      // x w first, then the two broadcast terms: no FFMA2 here reads three
      // register pairs (those issue at ~65 % of the pipe rate against ~90 %
      // with a broadcast operand, profiles/r01/probe_ffma2_banks.txt);
      // +1.0 % cfg5, +1.2 % cfg3 (profiles/r01/den_bcast_ab.txt)
      const float2 den = fma2(bc(cb), sbc, fma2(bc(ca), sab[q], mul2(x, sac)));  // 2 den
      const float2 num = fma2(bc(T.x), f[q].mx, fma2(bc(T.y), f[q].my, fma2(bc(T.z), f[q].mz, bc(T.w))));  // 2 num
      if (k & 1) {
        // den and num sit in the same operand slot of both products, so the
        // operand reuse cache can serve them (+0.5 %, profiles/r01/cprod_order_ab.txt)
        const float2 D = fma2(d0[q], den, mul2(make_float2(-n0[q].x, -n0[q].y), num));
        const float2 N = fma2(n0[q], den, mul2(d0[q], num));
        acc[q] = atan_far3(acc[q], N, D);
      } else {
        n0[q] = num;
        d0[q] = den;
      }
      ra[q] = rb[q];
      rb[q] = rc;
      sab[q] = sbc;
    }
  }
}

// ---- near evaluator -------------------------------------------------------
// Exact subtile frame of a point pair: -(p - c) = m + l as a double-single
// (m = -fl(hx - c), l = -(TwoSum error + lx)); R = (v - c) + m + l then has
// one rounding relative to |R| (not to |p - c|), so near a surface every
// term is accurate to ~ulp of its own geometry. Together with the snapped,
// watertight subtile vertices (nm_set_surfaces) this keeps the fp32 sum over
// a closed surface at its winding number for points close to vertices and
// edges.
struct NearFrame {
  float2 mx, my, mz, lx, ly, lz;
};

__device__ __forceinline__ void two_sum_neg(float2 a, float b, float2 lo_in, float2& m, float2& l) {
  const float2 s = add2(a, bc(b));
  const float2 bp = add2(s, make_float2(-a.x, -a.y));
  const float2 ap = add2(s, make_float2(-bp.x, -bp.y));
  const float2 err = add2(add2(a, make_float2(-ap.x, -ap.y)), add2(bc(b), make_float2(-bp.x, -bp.y)));
  const float2 lo = add2(err, lo_in);
  m = make_float2(-s.x, -s.y);
  l = make_float2(-lo.x, -lo.y);
}

// hi/lo of the centred point pair and the subtile centre c -> exact frame
__device__ __forceinline__ NearFrame near_frame(float2 hx, float2 hy, float2 hz, float2 lx, float2 ly, float2 lz,
                                                const float4& c) {
  NearFrame f;
  two_sum_neg(hx, -c.x, lx, f.mx, f.lx);
  two_sum_neg(hy, -c.y, ly, f.my, f.ly);
  two_sum_neg(hz, -c.z, lz, f.mz, f.lz);
  return f;
}

struct Vtx2 {
  float2 x, y, z, r;
};

// V holds 2V: R = (0.5 (2V) + m) + l, exact scaling, two roundings relative to |R|.
__device__ __forceinline__ Vtx2 strip_vertex(const float4& V, const NearFrame& f) {
  Vtx2 v;
  v.x = add2(fma2(bc(V.x), bc(0.5f), f.mx), f.lx);
  v.y = add2(fma2(bc(V.y), bc(0.5f), f.my), f.ly);
  v.z = add2(fma2(bc(V.z), bc(0.5f), f.mz), f.lz);
  const float2 q = fma2(v.z, v.z, fma2(v.y, v.y, mul2(v.x, v.x)));
  v.r = make_float2(sqrt_approx(q.x), sqrt_approx(q.y));
  return v;
}
__device__ __forceinline__ float2 dot2(const Vtx2& a, const Vtx2& b) {
  return fma2(a.z, b.z, fma2(a.y, b.y, mul2(a.x, b.x)));
}

#ifndef NM_NEAR_UNROLL
#define NM_NEAR_UNROLL 4
#endif
constexpr int kNearUnroll = NM_NEAR_UNROLL;
template <int NP>
__device__ __forceinline__ void seg_far(const float4* __restrict__ rec, const PairFrame (&f)[NP], float2 (&acc)[NP]) {
  float2 ra[NP], rb[NP], sab[NP];
  seg_far<NP>(rec, f, acc, ra, rb, sab, false);
}

// Near evaluator: R-based VOS terms with direct dot products (no
// |R_a|^2 + |R_b|^2 - |e|^2 identity, whose O(|e|^2) cancellation would cost
// ~eps |e| / r relative near a vertex), 3-term series for |x| <= kFarX, else
// the full-range atan2, plus the near-surface detector.
// use[k]: lane point k takes this group's near result (the caller discards
// the others), so only those lanes ask for the full-range atan2.
template <int NP>
__device__ __forceinline__ void seg_near(const float4* __restrict__ rec, const NearFrame (&f)[NP], float2 (&acc)[NP],
                                         bool (&det)[2 * NP], const bool (&use)[2 * NP], float tau, float delta) {
  Vtx2 a[NP], b[NP];
  float2 dab[NP];
  {
    const float4 V0 = rec[0], V1 = rec[1];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      a[q] = strip_vertex(V0, f[q]);
      b[q] = strip_vertex(V1, f[q]);
      dab[q] = dot2(a[q], b[q]);
    }
  }
#pragma unroll kNearUnroll
  for (int k = 0; k < kSegTris; ++k) {
    const float4 V2 = rec[k + 2];
    const float4 T = rec[kSegT + k];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const Vtx2 c = strip_vertex(V2, f[q]);
      const float2 dbc = dot2(b[q], c);
      const float2 dac = dot2(a[q], c);
      float2 num = fma2(bc(T.z), a[q].z, fma2(bc(T.y), a[q].y, mul2(bc(T.x), a[q].x)));
      num = mul2(num, bc(1.0f / kRecScale));  // exact: the record holds 2N
      const float2 den = fma2(fma2(a[q].r, b[q].r, dab[q]), c.r, fma2(dac, b[q].r, mul2(dbc, a[q].r)));
      const float2 af = acc_far2(acc[q], num, den);
      // |x| <= kFarX with den > 0: the 3-term series (af) is exact to fp32
      const bool frx = (den.x > 0.0f) && (fabsf(num.x) <= __fmul_rn(kFarX, den.x));
      const bool fry = (den.y > 0.0f) && (fabsf(num.y) <= __fmul_rn(kFarX, den.y));
      // near-surface detector
      const float2 lim = mul2(bc(tau), mul2(mul2(a[q].r, b[q].r), c.r));
      det[2 * q] |= ((fabsf(num.x) <= lim.x) && (den.x <= lim.x)) || (fminf(a[q].r.x, fminf(b[q].r.x, c.r.x)) <= delta);
      det[2 * q + 1] |=
          ((fabsf(num.y) <= lim.y) && (den.y <= lim.y)) || (fminf(a[q].r.y, fminf(b[q].r.y, c.r.y)) <= delta);
      // full-range atan2 only when some used lane of the warp needs it
      // (warp-uniform branch; a lane's value never depends on the others)
      float2 full = acc[q];
      if (__any_sync(0xffffffffu, (use[2 * q] && !frx) || (use[2 * q + 1] && !fry))) {
        full.x = __fadd_rn(acc[q].x, atan2_near(num.x, den.x));
        full.y = __fadd_rn(acc[q].y, atan2_near(num.y, den.y));
      }
      acc[q].x = frx ? af.x : full.x;
      acc[q].y = fry ? af.y : full.y;
      a[q] = b[q];
      b[q] = c;
      dab[q] = dbc;
    }
  }
}

// ---------------------------------------------------------------------------
// fp64 restatement for the fix-up pass: the operand order of the CPU oracle
// (vec3.hpp:32-38 dot/cross/norm, no FMA contraction), so a flagged pair's
// term differs from the oracle's only through atan2's last-ulp behaviour.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dot64(double ax, double ay, double az, double bx, double by, double bz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(ax, bx), __dmul_rn(ay, by)), __dmul_rn(az, bz));
}

__device__ __forceinline__ double vos_half_angle64(const double* a, const double* b, const double* c, double px,
                                                   double py, double pz, double* num_out = nullptr) {
  const double x1 = __dsub_rn(a[0], px), y1 = __dsub_rn(a[1], py), z1 = __dsub_rn(a[2], pz);
  const double x2 = __dsub_rn(b[0], px), y2 = __dsub_rn(b[1], py), z2 = __dsub_rn(b[2], pz);
  const double x3 = __dsub_rn(c[0], px), y3 = __dsub_rn(c[1], py), z3 = __dsub_rn(c[2], pz);
  const double l1 = __dsqrt_rn(dot64(x1, y1, z1, x1, y1, z1));
  const double l2 = __dsqrt_rn(dot64(x2, y2, z2, x2, y2, z2));
  const double l3 = __dsqrt_rn(dot64(x3, y3, z3, x3, y3, z3));
  // cross(R2, R3)
  const double cx = __dsub_rn(__dmul_rn(y2, z3), __dmul_rn(z2, y3));
  const double cy = __dsub_rn(__dmul_rn(z2, x3), __dmul_rn(x2, z3));
  const double cz = __dsub_rn(__dmul_rn(x2, y3), __dmul_rn(y2, x3));
  const double num = dot64(x1, y1, z1, cx, cy, cz);
  double den = __dmul_rn(__dmul_rn(l1, l2), l3);
  den = __dadd_rn(den, __dmul_rn(dot64(x1, y1, z1, x2, y2, z2), l3));
  den = __dadd_rn(den, __dmul_rn(dot64(x1, y1, z1, x3, y3, z3), l2));
  den = __dadd_rn(den, __dmul_rn(dot64(x2, y2, z2, x3, y3, z3), l1));
  if (num_out) *num_out = num;
  return atan2(num, den);
}


}  // namespace nm
