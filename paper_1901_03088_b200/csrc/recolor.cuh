// recolor.cuh — the per-lane recolour of one 48-byte block (16 pixels) in
// shared memory, shared by the single-slide kernel (xform.cu) and the batch
// kernel (batch.cu).
//
// OD table layouts in shared memory (REP replicas, so a warp's 32 lookups hit
// distinct banks):
//   REP 16: 64 KiB, rows of 256 B = [ch0 x16 | ch1 x16 | ch2 x16 | pad], copy
//           (lane&15) of channel c at x*256 + c*64 + (lane&15)*4 (<= 2-way
//           bank conflicts);
//   REP 24: 64 KiB, rows of 256 B = [ch0 x32 | ch1 x16 | ch2 x16]: channel 0
//           conflict-free (copy `lane`), channels 1 and 2 as REP 16 — 5 instead
//           of 6 shared-memory wavefronts per pixel's three lookups;
//   REP 32: 128 KiB, region 0 rows [ch0 x32 | ch1 x32], region 1 (+64 KiB)
//           rows [ch2 x32 | pad], copy `lane` at x*256 + ... + lane*4
//           (conflict-free).
// Either way ONE PRMT of (input word, per-lane constant) forms the address:
// byte 0 = the constant's low byte, byte 1 = the pixel byte x, byte 2 = the
// constant's region byte.
#pragma once
#include "spcn_device.cuh"

namespace spcn {

template <int REP>
struct LutLayout {
  static_assert(REP == 16 || REP == 24 || REP == 32,
                "table layouts exist for 16, 24 (mixed) and 32 replicas");
  static constexpr int kBytes = REP == 32 ? 2 * 65536 : 65536;

  // cooperative fill from a [3][256] fp32 table (any address space)
  __device__ static void fill(uint8_t* smem, const float* t, int tid, int nthreads) {
    if (REP == 24) {
      // rows of 256 B = [ch0 x32 | ch1 x16 | ch2 x16]
      for (int i = tid; i < 256 * 64; i += nthreads) {
        const int x = i >> 6, r = i & 63;
        const int c = r < 32 ? 0 : (r < 48 ? 1 : 2);
        *reinterpret_cast<float*>(smem + x * 256 + r * 4) = t[c * 256 + x];
      }
    } else if (REP == 16) {
      for (int i = tid; i < 256 * 48; i += nthreads) {
        const int x = i / 48, rem = i - 48 * x, c = rem >> 4, r = rem & 15;
        *reinterpret_cast<float*>(smem + x * 256 + c * 64 + r * 4) = t[c * 256 + x];
      }
    } else {
      for (int i = tid; i < 256 * 96; i += nthreads) {
        const int x = i / 96, rem = i - 96 * x, c = rem >> 5, r = rem & 31;
        const int off = (c == 2 ? 65536 : 0) + x * 256 + (c == 1 ? 128 : 0) + r * 4;
        *reinterpret_cast<float*>(smem + off) = t[c * 256 + x];
      }
    }
  }

  // per-lane PRMT constants of the three channels
  __device__ static void lane_consts(int lane, uint32_t (&lc)[3]) {
    if (REP == 24) {
      const uint32_t lrep = (uint32_t)(lane & 15) * 4;
      lc[0] = (uint32_t)lane * 4; lc[1] = 128u + lrep; lc[2] = 192u + lrep;
    } else if (REP == 16) {
      const uint32_t lrep = (uint32_t)(lane & 15) * 4;
      lc[0] = lrep; lc[1] = 64u + lrep; lc[2] = 128u + lrep;
    } else {
      const uint32_t lrep = (uint32_t)lane * 4;
      lc[0] = lrep; lc[1] = 128u + lrep; lc[2] = 0x10000u | lrep;
    }
  }
};

// (a ^ b) | c as a single LOP3 (opaque to the optimiser, which would otherwise
// turn the XOR into compare-and-select chains).
__device__ __forceinline__ uint32_t lop3_xor_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xBE;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// acc |= BIT if any of the three (lo, hi) float pairs differ: each pair is
// reinterpreted as one 64-bit float (its register pair, no moves) and
// compared with DSETP (fp64 pipe); the compares chain through one predicate
// that guards a single OR.
__device__ __forceinline__ double as_f64(float2 v) {
  union {
    float2 f;
    double d;
  } u;
  u.f = v;
  return u.d;
}
__device__ __forceinline__ void or_if_pairs_differ(uint32_t& acc, uint32_t bit,
                                                   const float2 (&lo)[3], const float2 (&hi)[3]) {
  asm("{\n\t.reg .pred p;\n\t"
      "setp.neu.f64 p, %1, %2;\n\t"
      "setp.neu.or.f64 p, %3, %4, p;\n\t"
      "setp.neu.or.f64 p, %5, %6, p;\n\t"
      "@p or.b32 %0, %0, %7;\n\t}"
      : "+r"(acc)
      : "d"(as_f64(lo[0])), "d"(as_f64(hi[0])), "d"(as_f64(lo[1])), "d"(as_f64(hi[1])),
        "d"(as_f64(lo[2])), "d"(as_f64(hi[2])), "r"(bit));
}

// OD of input byte `idx` (0..47) of the thread's 48-byte block, channel c.
// ABS != 0: the table sits at the absolute shared-memory address ABS (the
// caller placed it there), and `lut` is unused — the load is LDS [addr+ABS],
// with no shared-window base to keep in a register.
template <int ABS = 0>
__device__ __forceinline__ float od_lookup(const uint8_t* lut, const uint32_t* w, int idx,
                                           uint32_t lc) {
  const uint32_t sel = 0x7604u | ((uint32_t)(idx & 3) << 4);
  const uint32_t addr = __byte_perm(w[idx >> 2], lc, sel);  // region*64K + x*256 + low byte
  if constexpr (ABS != 0) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(ABS));
    return v;
  } else {
    return *reinterpret_cast<const float*>(lut + addr);
  }
}

__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// Recolor two pixels (k, k+1) of the block; writes their 6 output "bytes"
// (low byte of each word) to ob[3k .. 3k+5].  MODE 0 = EXACT (analytic
// per-pixel bound), 1 = FAST, 2 = EXACT (calibrated constant bound).  EXACT:
// returns non-zero when any of the pair's six roundings is not certified
// (r_lo != r_hi); both pixels of such a pair go to the fp64 repair list.
// I: the calibrated {I_lo, I_hi} per channel (MODE 2).
template <int MODE, int ABS = 0>
__device__ __forceinline__ uint32_t recolor_pair(const FastS& fp, const uint8_t* lut,
                                                 const uint32_t* w, int k, const uint32_t* lc,
                                                 uint32_t* ob, const float2* I,
                                                 uint32_t* badpairs = nullptr) {
  const int a = 3 * k, b = 3 * k + 3;
  const float2 v0 =
      make_float2(od_lookup<ABS>(lut, w, a, lc[0]), od_lookup<ABS>(lut, w, b, lc[0]));
  const float2 v1 =
      make_float2(od_lookup<ABS>(lut, w, a + 1, lc[1]), od_lookup<ABS>(lut, w, b + 1, lc[1]));
  const float2 v2 =
      make_float2(od_lookup<ABS>(lut, w, a + 2, lc[2]), od_lookup<ABS>(lut, w, b + 2, lc[2]));
  const FastPair fq = fast_pair(fp, v0, v1, v2);
  const float e[3][2] = {{fq.e0.x, fq.e0.y}, {fq.e1.x, fq.e1.y}, {fq.e2.x, fq.e2.y}};
  if (MODE == 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float2 pw = make_float2(ex2_approx(e[c][0]), ex2_approx(e[c][1]));
      const float2 r = __ffma2_rn(bc2(fp.i0t[c]), pw, bc2(kMagic));
      ob[a + c] = __float_as_uint(r.x);
      ob[b + c] = __float_as_uint(r.y);
    }
    return 0u;
  }
  if (MODE == 2) {
    // calibrated constant interval: {lo, hi} of BOTH pixels of the pair in two
    // FFMA2 (pixel pair x one interval end), and the certification test of
    // the pair's six roundings as three 64-bit compares of (lo_a, lo_b) with
    // (hi_a, hi_b) accumulated in one predicate (DSETP on the fp64 pipe, off
    // the saturated ALU/FMA issue).  Magic-number floats are never NaN or
    // zero, so 64-bit float inequality is bit inequality.
    float2 lo[3], hi[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float2 pw = make_float2(ex2_approx(e[c][0]), ex2_approx(e[c][1]));
      lo[c] = __ffma2_rn(bc2(I[c].x), pw, bc2(kMagic));
      hi[c] = __ffma2_rn(bc2(I[c].y), pw, bc2(kMagic));
      ob[a + c] = __float_as_uint(hi[c].x);
      ob[b + c] = __float_as_uint(hi[c].y);
    }
    or_if_pairs_differ(*badpairs, 1u << (k >> 1), lo, hi);
    return 0u;
  }
  if (MODE == 0) {
    // analytic per-pixel bound: alpha of both pixels in one FFMA2, then per
    // channel the interval ends of BOTH pixels (lo pair, hi pair: two FFMA2.RD
    // with the same element operations as cert_interval), their roundings in
    // two FFMA2 and the compare as in MODE 2 (no per-pixel operand shuffles)
    const float2 alpha = __ffma2_rn(bc2(fp.a1), fq.T, bc2(fp.a0));
    float2 lo[3], hi[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float2 pw = make_float2(ex2_approx(e[c][0]), ex2_approx(e[c][1]));
      const float2 ilo = __ffma2_rd(bc2(-fp.i0t[c]), alpha, bc2(fp.i0t[c]));
      const float2 ihi = __ffma2_rd(bc2(fp.i0t[c]), alpha, bc2(fp.i0t[c]));
      lo[c] = __ffma2_rn(ilo, pw, bc2(kMagic));
      hi[c] = __ffma2_rn(ihi, pw, bc2(kMagic));
      ob[a + c] = __float_as_uint(hi[c].x);
      ob[b + c] = __float_as_uint(hi[c].y);
    }
    uint32_t bad = 0;
    or_if_pairs_differ(bad, 1u, lo, hi);
    return bad;
  }
  float2 alpha = bc2(0.f);
  uint32_t bad = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float pa = ex2_approx(e[c][0]), pb = ex2_approx(e[c][1]);
    float2 Ia, Ib;
    if (MODE == 0) {
      Ia = cert_interval(fp.i0t[c], alpha.x);
      Ib = cert_interval(fp.i0t[c], alpha.y);
    } else {
      Ia = Ib = I[c];
    }
    const float2 ra = __ffma2_rn(Ia, bc2(pa), bc2(kMagic));
    const float2 rb = __ffma2_rn(Ib, bc2(pb), bc2(kMagic));
    ob[a + c] = __float_as_uint(ra.y);
    ob[b + c] = __float_as_uint(rb.y);
    bad = lop3_xor_or(__float_as_uint(ra.y), __float_as_uint(ra.x), bad);   // one LOP3 each
    bad = lop3_xor_or(__float_as_uint(rb.y), __float_as_uint(rb.x), bad);
  }
  return bad;
}

// One lane's 16 pixels at `blk` (48 bytes in shared memory), recoloured in
// place; `gp0` = global index of its first pixel.  MODE 3 = identity copy
// (memory-path ceiling).  Whole warp calls (the repair append is warp-wide).
template <int MODE, int ABS = 0>
__device__ __forceinline__ void recolor_block(const FastS& fp, const uint8_t* lut,
                                              const uint32_t* lc, uint8_t* blk, bool valid,
                                              int64_t gp0, const RepairList& rl, int lane,
                                              const float2* I) {
  uint32_t w[12], ob[48], o[12];
  uint32_t badpairs = 0;
  if (valid) {
    const uint4* q = reinterpret_cast<const uint4*>(blk);
    const uint4 q0 = q[0], q1 = q[1], q2 = q[2];
    w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w;
    w[4] = q1.x; w[5] = q1.y; w[6] = q1.z; w[7] = q1.w;
    w[8] = q2.x; w[9] = q2.y; w[10] = q2.z; w[11] = q2.w;
  }
  if (MODE != 3 && fp.wmask) {
    // background blocks (every byte >= the OD-zero threshold) render the
    // constant target background; skip the math when the whole warp has them
    // (two stages: the first 4 pixels of every lane, then the rest — tissue
    // warps leave after one LOP3 and one vote)
    uint32_t acc = valid ? (w[0] & w[1] & w[2]) : 0xffffffffu;
    bool bg = __all_sync(0xffffffffu, (acc & fp.wmask) == fp.wmask);
    if (bg) {
      if (valid) {
#pragma unroll
        for (int t = 3; t < 12; ++t) acc &= w[t];
      }
      bg = __all_sync(0xffffffffu, (acc & fp.wmask) == fp.wmask);
    }
    if (bg) {
      if (valid) {
        uint4* d = reinterpret_cast<uint4*>(blk);
        d[0] = make_uint4(fp.wout[0], fp.wout[1], fp.wout[2], fp.wout[0]);
        d[1] = make_uint4(fp.wout[1], fp.wout[2], fp.wout[0], fp.wout[1]);
        d[2] = make_uint4(fp.wout[2], fp.wout[0], fp.wout[1], fp.wout[2]);
      }
      return;
    }
  }
  if (valid) {
    if (MODE == 3) {
#pragma unroll
      for (int t = 0; t < 12; ++t) o[t] = w[t];
    } else {
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        const uint32_t bad = recolor_pair<MODE, ABS>(fp, lut, w, 2 * qq, lc, ob, I, &badpairs);
        if (MODE == 0) badpairs |= (bad != 0u ? 1u : 0u) << qq;
#pragma unroll
        for (int t = 0; t < 12; ++t)
          if (4 * t + 3 >= 6 * qq && 4 * t + 3 < 6 * qq + 6)
            o[t] = pack4(ob[4 * t], ob[4 * t + 1], ob[4 * t + 2], ob[4 * t + 3]);
      }
    }
  }
  if ((MODE == 0 || MODE == 2) && __any_sync(0xffffffffu, badpairs != 0u))
    repair_append(badpairs, blk, gp0, rl.count, rl.items, rl.cap, lane);
  if (valid) {   // output in place over the (already consumed) input block
    uint4* d = reinterpret_cast<uint4*>(blk);
    d[0] = make_uint4(o[0], o[1], o[2], o[3]);
    d[1] = make_uint4(o[4], o[5], o[6], o[7]);
    d[2] = make_uint4(o[8], o[9], o[10], o[11]);
  }
}

}  // namespace spcn
