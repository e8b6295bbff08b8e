// Compact register-machine interpreter for fused elementwise programs
// (shared by the elementwise and reduction kernels).
//
// The program (spx_insn[], in kernel-parameter constant memory) is uniform
// across the grid, so every branch below is warp-uniform.  Slot reads and
// writes are `switch`es over compile-time slots: the SPX_NREG-value register
// file lives in registers, and the loop over instructions is NOT unrolled --
// a first version that unrolled it thrashed the instruction cache (ncu:
// 56% of stalls "no_instruction").
#pragma once
#include "common.cuh"

template <int W>
struct Vec {
  float v[W];
};

template <int W>
struct RegFile {
  Vec<W> r[SPX_NREG];

  SPX_DEV Vec<W> get(int i) const {
    switch (i) {
#define SPX_GET(k) case k: return r[k];
      SPX_GET(0) SPX_GET(1) SPX_GET(2) SPX_GET(3) SPX_GET(4) SPX_GET(5)
      SPX_GET(6) SPX_GET(7) SPX_GET(8) SPX_GET(9) SPX_GET(10) SPX_GET(11)
#undef SPX_GET
    }
    return r[0];
  }
  SPX_DEV void set(int i, const Vec<W>& x) {
    switch (i) {
#define SPX_SET(k) case k: r[k] = x; break;
      SPX_SET(0) SPX_SET(1) SPX_SET(2) SPX_SET(3) SPX_SET(4) SPX_SET(5)
      SPX_SET(6) SPX_SET(7) SPX_SET(8) SPX_SET(9) SPX_SET(10) SPX_SET(11)
#undef SPX_SET
    }
  }
};

template <int W>
SPX_DEV void run_program(const spx_insn* prog, const float* imm, int n, RegFile<W>& f) {
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    const spx_insn in = prog[i];
    const float c = imm[i];
    const Vec<W> a = f.get(in.a);
    Vec<W> y;
    switch (in.op) {
      case SPX_OP_ADD: { const Vec<W> b = f.get(in.b);
#pragma unroll
        for (int k = 0; k < W; ++k) y.v[k] = f_add(a.v[k], b.v[k]);
        break; }
      case SPX_OP_MUL: { const Vec<W> b = f.get(in.b);
#pragma unroll
        for (int k = 0; k < W; ++k) y.v[k] = f_mul(a.v[k], b.v[k]);
        break; }
      case SPX_OP_MAX: { const Vec<W> b = f.get(in.b);
#pragma unroll
        for (int k = 0; k < W; ++k) y.v[k] = f_max(a.v[k], b.v[k]);
        break; }
      default:
#pragma unroll
        for (int k = 0; k < W; ++k) y.v[k] = apply_op(in.op, a.v[k], 0.f, c);
    }
    f.set(in.dst, y);
  }
}
