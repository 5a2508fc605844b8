// smem_merge.cuh — shared-memory merge levels with sentinel-terminated runs.
//
// One level merges runs pairwise (run 2q with run 2q+1) from buffer X into
// buffer Y.  Every input run is followed by a +inf sentinel, so the merge loop
// has no bounds tests (the merge_runs loop of hybrid.hpp:69-76 without its
// `i < left_len && j <= right` checks).  The CTA's threads split the level's
// concatenated output by position; thread t starts at
//     d_t = t*Kb + 2*((t >> 2) & 7)
// — the skew term puts the merge cursors of the 32 lanes of a warp (≈ d_t/2
// into each run) on 32 different banks even when Kb is a multiple of 16, so
// the layout needs no padding words and no per-access index arithmetic.
#pragma once
#include <climits>
#include <cstdint>

namespace nsb {

constexpr int kMaxRuns = 16;

struct RunSet {  // lives in shared memory
  int n;
  int off[kMaxRuns];
  int len[kMaxRuns];
  __device__ __forceinline__ int count() const { return n; }
  __device__ __forceinline__ int offset(int r) const { return off[r]; }
  __device__ __forceinline__ int length(int r) const { return len[r]; }
};

// n equal runs of length `len` laid out every `stride` words.
struct RegularRuns {
  int n, len, stride;
  __device__ __forceinline__ int count() const { return n; }
  __device__ __forceinline__ int offset(int r) const { return r * stride; }
  __device__ __forceinline__ int length(int) const { return len; }
};

__device__ __forceinline__ int skew_diag(int t, int kb, int total) {
  return min(total, t * kb + 2 * ((t >> 2) & 7));
}

// Merge-path split on sentinel runs (A wins ties).
__device__ __forceinline__ int smem_merge_path(const int32_t* A, int a_len, const int32_t* B,
                                               int b_len, int diag) {
  int lo = max(0, diag - b_len), hi = min(diag, a_len);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A[mid] <= B[diag - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Emits `cnt` merged keys starting at (A+a, B+b) into Y[0..cnt).  Within one
// thread the tie rule does not change the emitted values (keys only), so the
// loop is branch-free: out = min(ka, kb), advance the side that held it and
// reload ONLY that side (one LDS per key: the data-dependent LDS is the
// bank-conflicted access, so it is the one to minimise).  PTX on 32-bit
// shared-memory byte addresses; per key 1 LDS + 1 STS + 2 ISETP + 1 IMNMX +
// 1 SEL + 2 predicated IADD + 2 predicated MOV.  A is never stepped past its
// sentinel: when ka == +inf both heads are +inf and so is every remaining
// output; take_a false implies kb < ka, so B cannot pass its sentinel either.
#ifdef NSB_DEBUG_KWAY
__device__ int g_dbg[8];
__device__ __forceinline__ void dbg_record(int code, int x, int y, int z) {
  if (atomicCAS(&g_dbg[0], 0, code) == 0) {
    g_dbg[1] = x;
    g_dbg[2] = y;
    g_dbg[3] = z;
    g_dbg[4] = blockIdx.x;
    g_dbg[5] = threadIdx.x;
  }
}
#endif

__device__ __forceinline__ void sentinel_merge(const int32_t* A, const int32_t* B, int a, int b,
                                               int32_t* Y, int cnt) {
#ifdef NSB_DEBUG_KWAY
  {
    extern __shared__ int32_t kw_sm[];
    const int lim = 2 * (7936 + 64 + 16);
    const int ia = (int)(A + a - kw_sm), ib = (int)(B + b - kw_sm), iy = (int)(Y - kw_sm);
    if (ia < 0 || ia >= lim || ib < 0 || ib >= lim || iy < 0 || iy + cnt > lim || cnt < 0) {
      dbg_record(1, ia, ib, iy * 100000 + cnt);
      return;
    }
    const int32_t* pa = A + a;
    const int32_t* pb = B + b;
    for (int k = 0; k < cnt; ++k) {
      const int ja = (int)(pa - kw_sm), jb = (int)(pb - kw_sm);
      if (ja < 0 || ja >= lim || jb < 0 || jb >= lim) {
        dbg_record(2, ja, jb, k);
        return;
      }
      const int32_t ka = *pa, kb = *pb;
      const bool take_a = ka <= kb;
      Y[k] = take_a ? ka : kb;
      pa += take_a & (ka != INT_MAX);
      pb += !take_a;
    }
    return;
  }
#endif
  uint32_t pa = static_cast<uint32_t>(__cvta_generic_to_shared(A + a));
  uint32_t pb = static_cast<uint32_t>(__cvta_generic_to_shared(B + b));
  uint32_t py = static_cast<uint32_t>(__cvta_generic_to_shared(Y));
  const uint32_t py_end = py + 4u * (uint32_t)cnt;
  int32_t ka, kb;
  asm volatile("ld.shared.b32 %0, [%2];\n ld.shared.b32 %1, [%3];\n"
               : "=&r"(ka), "=&r"(kb)
               : "r"(pa), "r"(pb)
               : "memory");
#pragma unroll 1
  for (; py + 16u <= py_end; py += 16u) {
    asm volatile(
        "{\n"
        " .reg .b32 o, ad, x;\n"
        " .reg .pred p, q;\n"
        " setp.le.s32 p, %2, %3;\n"
        " min.s32 o, %2, %3;\n"
        " st.shared.b32 [%4+0], o;\n"
        " setp.ne.and.s32 q, %2, 0x7fffffff, p;\n"
        " @q add.u32 %0, %0, 4;\n"
        " @!p add.u32 %1, %1, 4;\n"
        " selp.b32 ad, %0, %1, p;\n"
        " ld.shared.b32 x, [ad];\n"
        " @p mov.b32 %2, x;\n"
        " @!p mov.b32 %3, x;\n"
        " setp.le.s32 p, %2, %3;\n"
        " min.s32 o, %2, %3;\n"
        " st.shared.b32 [%4+4], o;\n"
        " setp.ne.and.s32 q, %2, 0x7fffffff, p;\n"
        " @q add.u32 %0, %0, 4;\n"
        " @!p add.u32 %1, %1, 4;\n"
        " selp.b32 ad, %0, %1, p;\n"
        " ld.shared.b32 x, [ad];\n"
        " @p mov.b32 %2, x;\n"
        " @!p mov.b32 %3, x;\n"
        " setp.le.s32 p, %2, %3;\n"
        " min.s32 o, %2, %3;\n"
        " st.shared.b32 [%4+8], o;\n"
        " setp.ne.and.s32 q, %2, 0x7fffffff, p;\n"
        " @q add.u32 %0, %0, 4;\n"
        " @!p add.u32 %1, %1, 4;\n"
        " selp.b32 ad, %0, %1, p;\n"
        " ld.shared.b32 x, [ad];\n"
        " @p mov.b32 %2, x;\n"
        " @!p mov.b32 %3, x;\n"
        " setp.le.s32 p, %2, %3;\n"
        " min.s32 o, %2, %3;\n"
        " st.shared.b32 [%4+12], o;\n"
        " setp.ne.and.s32 q, %2, 0x7fffffff, p;\n"
        " @q add.u32 %0, %0, 4;\n"
        " @!p add.u32 %1, %1, 4;\n"
        " selp.b32 ad, %0, %1, p;\n"
        " ld.shared.b32 x, [ad];\n"
        " @p mov.b32 %2, x;\n"
        " @!p mov.b32 %3, x;\n"
        "}\n"
        : "+r"(pa), "+r"(pb), "+r"(ka), "+r"(kb)
        : "r"(py)
        : "memory");
  }
#pragma unroll 1
  for (; py < py_end; py += 4u) {
    asm volatile(
        "{\n"
        " .reg .b32 o, ad, x;\n"
        " .reg .pred p, q;\n"
        " setp.le.s32 p, %2, %3;\n"
        " min.s32 o, %2, %3;\n"
        " st.shared.b32 [%4+0], o;\n"
        " setp.ne.and.s32 q, %2, 0x7fffffff, p;\n"
        " @q add.u32 %0, %0, 4;\n"
        " @!p add.u32 %1, %1, 4;\n"
        " selp.b32 ad, %0, %1, p;\n"
        " ld.shared.b32 x, [ad];\n"
        " @p mov.b32 %2, x;\n"
        " @!p mov.b32 %3, x;\n"
        "}\n"
        : "+r"(pa), "+r"(pb), "+r"(ka), "+r"(kb)
        : "r"(py)
        : "memory");
  }
}

// One pairwise level: X runs `in` -> Y runs `out` (out.length(q) ==
// in.length(2q) + in.length(2q+1)).  If `sentinels`, a +inf is written after
// every output run.  Caller synchronises before and after.
template <int NT, class IN, class OUT>
__device__ __forceinline__ void merge_level(const int32_t* X, const IN& in, int32_t* Y,
                                            const OUT& out, int total, bool sentinels,
                                            int min_kb = 1) {
  const int tid = threadIdx.x;
  if (sentinels && tid < out.count()) Y[out.offset(tid) + out.length(tid)] = INT_MAX;
  // odd outputs per thread: lanes' STS and merge cursors land on distinct
  // banks; min_kb > NT/total concentrates the work on fewer threads so each
  // merge-path search is amortised over more outputs
  const int kb = max((total + NT - 1) / NT, min_kb) | 1;
  int pos = min(total, tid * kb);
  const int end = min(total, (tid + 1) * kb);
  // locate the output run holding `pos`
  int q = 0, qbase = 0;
  while (q + 1 < out.count() && pos >= qbase + out.length(q)) {
    qbase += out.length(q);
    ++q;
  }
  while (pos < end) {
    const int qlen = out.length(q);
    const int seg_end = min(end, qbase + qlen);
    const int diag = pos - qbase;
    const int ra = 2 * q, rb = 2 * q + 1;
    const int32_t* A = X + in.offset(ra);
    const int a_len = in.length(ra);
    const bool has_b = rb < in.count();
    const int32_t* B = has_b ? X + in.offset(rb) : A + a_len;  // sentinel acts as an empty run
    const int b_len = has_b ? in.length(rb) : 0;
    const int a = smem_merge_path(A, a_len, B, b_len, diag);
    sentinel_merge(A, B, a, diag - a, Y + out.offset(q) + diag, seg_end - pos);
    pos = seg_end;
    qbase += qlen;
    ++q;
  }
}

}  // namespace nsb
