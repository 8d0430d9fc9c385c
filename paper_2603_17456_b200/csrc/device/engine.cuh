// Device-resident event loop of the flow-level simulator: one warp owns one
// simulation instance and runs its whole event loop without host round trips.
//
// Per processed event (Engine::run, engine.cpp:595-657):
//   K4  next-event selection: warp argmin over (t, klass, seq) of the arrival
//       stream head, the small non-flow event pool and the per-active-flow
//       completion slots (replaces std::priority_queue + stale generations);
//       streaming `advance_to` over the active SoA (engine.cpp:261-276)
//   K1  stage-DAG release / admission handlers (engine.cpp:295-593)
//   K2  RMLQ promotion (rmlq.cpp:101-193, allocator.cpp:128-171)
//   K3  class construction per policy (baselines.cpp:23-135, rmlq.cpp:201-260)
//       and strict-priority progressive filling (allocator.cpp:28-126)
//   K5  MFS Algorithm 1 at batch events (rmlq.cpp:268-382, inter_request.cpp)
//
// Exactness: every FP operation that the reference performs is performed here
// in the same order with IEEE double round-to-nearest and no contraction
// (built with -fmad=false; critical spots use __d*_rn explicitly). Decisions
// that the reference takes in container order (active_ swap-remove order,
// push seq numbering, unordered_map iteration in load_fraction) are replayed.
#pragma once
#include <math.h>
#include <stdint.h>
#if !defined(__CUDACC__)
#include <string.h>
#endif

#include "lanes.cuh"
#include "layout.h"

namespace mfb {

#define MF_INF (__builtin_huge_val())
constexpr double kNoTime = -1.0;
constexpr unsigned long long kNoSeq = ~0ull;

// libstdc++ _Prime_rehash_policy schedule for an unordered_map grown one
// insertion at a time from empty (measured; see oracle/hash_schedule.cpp).
constexpr int kHashStages = 19;
#if defined(__CUDACC__)
__device__ __constant__ int kRehashAt[kHashStages] = {
#else
static const int kRehashAt[kHashStages] = {
#endif
    0,     13,     29,     59,     127,    257,    541,     1109,    2357,   5087,
    10273, 20753,  42043,  85229,  172933, 351061, 712697,  1447153, 2938679};
#if defined(__CUDACC__)
__device__ __constant__ int kBucketsAt[kHashStages] = {
#else
static const int kBucketsAt[kHashStages] = {
#endif
    13,    29,     59,     127,    257,    541,     1109,    2357,    5087,   10273,
    20753, 42043,  85229,  172933, 351061, 712697,  1447153, 2938679, 5967347};

// ---------------------------------------------------------------------------
// IEEE helpers (std::min / std::max argument-order semantics)

MF_FN double smin(double a, double b) { return (b < a) ? b : a; }
MF_FN double smax(double a, double b) { return (a < b) ? b : a; }
#if defined(__CUDACC__)
MF_FN double dmul(double a, double b) { return __dmul_rn(a, b); }
MF_FN double dadd(double a, double b) { return __dadd_rn(a, b); }
MF_FN double dsub(double a, double b) { return __dsub_rn(a, b); }
MF_FN double ddiv(double a, double b) { return __ddiv_rn(a, b); }
MF_FN unsigned long long dbits(double x) { return (unsigned long long)__double_as_longlong(x); }
MF_FN bool isnan_(double x) { return isnan(x); }
#else
MF_FN double dmul(double a, double b) { return a * b; }
MF_FN double dadd(double a, double b) { return a + b; }
MF_FN double dsub(double a, double b) { return a - b; }
MF_FN double ddiv(double a, double b) { return a / b; }
MF_FN unsigned long long dbits(double x) {
  unsigned long long u;
  memcpy(&u, &x, 8);
  return u;
}
MF_FN bool isnan_(double x) { return x != x; }
#endif
#if defined(__CUDACC__)
MF_FN unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#else
MF_FN unsigned long long now_ns() { return 0; }
#endif

#if defined(__CUDACC__)
MF_FN double bits_to_d(unsigned long long u) { return __longlong_as_double((long long)u); }
#else
MF_FN double bits_to_d(unsigned long long u) {
  double d;
  memcpy(&d, &u, 8);
  return d;
}
#endif
// order-preserving map double -> u64 (non-NaN; -0 folded onto +0)
MF_FN unsigned long long dord(double x) {
  if (x == 0.0) x = 0.0;
  unsigned long long u = dbits(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
#if defined(__CUDACC__)
MF_FN int ctz32(unsigned m) { return __ffs(m) - 1; }
MF_FN int popc32(unsigned m) { return __popc(m); }
#else
MF_FN int ctz32(unsigned m) { return __builtin_ctz(m); }
MF_FN int popc32(unsigned m) { return __builtin_popcount(m); }
#endif
// Tell the compiler a pointer addresses shared memory (LDS/STS/ATOMS instead
// of generic accesses) when the instance's hot arrays were staged on chip.
#if defined(__CUDACC__)
#define MF_SH(ptr) __builtin_assume(__isShared(ptr))
#else
#define MF_SH(ptr) ((void)0)
#endif

// 1/n correctly rounded for small n (exact table), else a division
#if defined(__CUDACC__)
__device__ __constant__ double kRecipTab[65] = {
#else
static const double kRecipTab[65] = {
#endif
    0.0,     1.0 / 1,  1.0 / 2,  1.0 / 3,  1.0 / 4,  1.0 / 5,  1.0 / 6,  1.0 / 7,  1.0 / 8,
    1.0 / 9,  1.0 / 10, 1.0 / 11, 1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15, 1.0 / 16, 1.0 / 17,
    1.0 / 18, 1.0 / 19, 1.0 / 20, 1.0 / 21, 1.0 / 22, 1.0 / 23, 1.0 / 24, 1.0 / 25, 1.0 / 26,
    1.0 / 27, 1.0 / 28, 1.0 / 29, 1.0 / 30, 1.0 / 31, 1.0 / 32, 1.0 / 33, 1.0 / 34, 1.0 / 35,
    1.0 / 36, 1.0 / 37, 1.0 / 38, 1.0 / 39, 1.0 / 40, 1.0 / 41, 1.0 / 42, 1.0 / 43, 1.0 / 44,
    1.0 / 45, 1.0 / 46, 1.0 / 47, 1.0 / 48, 1.0 / 49, 1.0 / 50, 1.0 / 51, 1.0 / 52, 1.0 / 53,
    1.0 / 54, 1.0 / 55, 1.0 / 56, 1.0 / 57, 1.0 / 58, 1.0 / 59, 1.0 / 60, 1.0 / 61, 1.0 / 62,
    1.0 / 63, 1.0 / 64};
MF_FN double recip(int n) { return n <= 64 ? kRecipTab[n] : ddiv(1.0, (double)n); }
#if defined(__CUDACC__)
MF_FN double frecip(int n) { return (double)__frcp_rn((float)n); }
#else
MF_FN double frecip(int n) { return (double)(1.0f / (float)n); }
#endif

MF_FN int klass_of(int kind) { return kind <= EV_DEPART ? 0 : (kind == EV_TICK ? 2 : 1); }
MF_FN int pow2ceil(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Scalar state: every lane keeps an identical register copy.
struct Sc {
  double now;
  double prev_t;
  double horizon;
  unsigned long long seq;
  long long events, steps, streak, pushes, algo_bytes, classes, rounds;
  long long stop_at;  // event count at which this launch suspends
  int pend_ncls;      // classes of a rate recomputation split over gang barriers (-1: none)
  int pend_kind, pend_a, pend_b;  // the popped event between step_head and step_dispatch
  bool pend_caps;
  int n_flows, n_batches, n_coflows, n_active, n_ev;
  int rp_top, pp_top, cm_top;
  int next_arr;
  unsigned epoch;
  int n_live;
  int h_n, h_ready;
  int n_srt, n_add;
  int sl_hw, sl_nfree, n_unslotted;
  bool bk_slots;
  int bk_n;
  bool rel_idx;
  int dirty;
  int err, chk;
  long long pruned;
  int max_active;
  int max_touch, max_pool;
  double sat_max;  // 1e-12 * the largest link capacity: bounds every saturation threshold
  long long cy[32];
};

#if defined(MF_PROF) && defined(__CUDACC__)
#define MF_TIC(v) long long v = clock64()
#define MF_RETIC(v) v = clock64()
#define MF_TOC(slot, v) s.cy[slot - OUT_CY_NEXT] += clock64() - v
#else
#define MF_TIC(v)
#define MF_RETIC(v)
#define MF_TOC(slot, v)
#endif

struct Ev {
  double t;
  int klass;
  unsigned long long seq;
  int src;  // 0 none, 1 arrival, 2 pool, 3 flow slot
  int idx;
};

MF_FN bool ev_less(const Ev& x, const Ev& y) {
  if (x.t != y.t) return x.t < y.t;
  if (x.klass != y.klass) return x.klass < y.klass;
  return x.seq < y.seq;
}

// One engine per warp. `chip`: the kernel staged the per-slot filling state
// and the frozen-member bits in shared memory (engine_kernel.cu make_plan);
// only the filling rounds are specialised on it, the rest of the engine is
// one copy of code (instruction-cache footprint).
// kAalo: the Aalo extension's code is compiled in (a separate kernel instance,
// launched only for batches holding aalo instances: the engine is
// instruction-fetch bound and every code byte counts, profiles/r01_ab_engine_builds.txt)
template <class G, bool kAalo = true>
struct Engine {
  G g;
  Inst& I;  // per-warp copy (shared memory on the device), arrays possibly re-pointed
  bool chip;
  Sc s;

  MF_FN explicit Engine(Inst& inst, bool on_chip = false) : I(inst), chip(on_chip) {}

  // ----------------------------------------------------------------- util
  template <class T>
  MF_FN void put(T* p, T v) { g.put(p, v); }
  MF_FN void fail(int code, int chk) {
    if (!s.err) {
      s.err = code;
      s.chk = chk;
    }
  }
  MF_FN int rbeg(int fid) const {
    const int r = I.f_route[fid];
    return r >= 0 ? I.route_off[r] : 0;
  }
  MF_FN int rlen(int fid) const {
    const int r = I.f_route[fid];
    return r >= 0 ? I.route_off[r + 1] - I.route_off[r] : 0;
  }
  MF_FN bool done(int fid) const { return I.f_state[fid] == FL_DONE; }
  // cached route of the active flow at position p
  MF_FN int arl(int p, int k) const { return I.a_rl[p * I.rmax + k]; }
  MF_FN int arn(int p) const { return I.a_rn[p]; }
  MF_FN double remaining(int fid) const {
    int p = I.f_apos[fid];
    if (p >= 0) return I.a_rem[p];
    return I.f_state[fid] == FL_DONE ? 0.0 : I.f_size[fid];
  }
  MF_FN bool has_dl(int fid) const { return !isnan_(I.f_dl[fid]); }
  MF_FN bool outranks(int ba, int la, int bb, int lb) const {
    if (ba != bb) return ba < bb;
    return la < lb;
  }

  // ------------------------------------------------------------ event pool
  MF_FN void push(double t, int kind, int a, int b) {
    if (s.n_ev >= I.E_cap) {
      fail(ERR_INTERNAL, CHK_CAP_EVENTS);
      return;
    }
    const int i = s.n_ev;
    g.sync();
    if (g.leader()) {
      I.e_t[i] = t;
      I.e_seq[i] = s.seq;
      I.e_kind[i] = kind;
      I.e_a[i] = a;
      I.e_b[i] = b;
    }
    g.sync();
    ++s.n_ev;
    ++s.seq;
    ++s.pushes;
    if (s.n_ev > s.max_pool) s.max_pool = s.n_ev;
  }

  // K4: the earliest of the arrival head, the event pool and the per-flow
  // completion slots under (t, klass, seq) (engine.hpp:182-188). klass and seq
  // share one 64-bit key (seq < 2^61); source and index share one int.
  MF_FN Ev next_event() {
    const int ne = s.n_ev, na = s.n_active;
    const double* __restrict__ et = I.e_t;
    const unsigned long long* __restrict__ es = I.e_seq;
    const int* __restrict__ ek = I.e_kind;
    const double* __restrict__ at = I.a_evt;
    const unsigned long long* __restrict__ as = I.a_evseq;
    double bt = MF_INF;
    unsigned long long bk = ~0ull;
    int bsi = 0;  // (src << 28) | idx, src 0 = none
    if (g.leader() && s.next_arr < I.n_arr) {
      const int r = I.arr_order[s.next_arr];
      bt = I.r_arrival[r];
      bk = (1ull << 61) | (unsigned long long)r;
      bsi = (1 << 28) | r;
    }
#pragma unroll 2
    for (int i = g.lane(); i < ne; i += G::N) {
      const double t = et[i];
      const unsigned long long k = ((unsigned long long)klass_of(ek[i]) << 61) | es[i];
      if (t < bt || (t == bt && k < bk)) {
        bt = t;
        bk = k;
        bsi = (2 << 28) | i;
      }
    }
MF_UNROLL
    for (int p = g.lane(); p < na; p += G::N) {
      const unsigned long long k = as[p];
      const double t = at[p];
      if (k != kNoSeq && (t < bt || (t == bt && k < bk))) {
        bt = t;
        bk = k;
        bsi = (3 << 28) | p;
      }
    }
    g.argmin_tk(&bt, &bk, &bsi);  // event times are >= 0 (or -0), never NaN
    Ev best;
    best.t = bt;
    best.klass = (int)(bk >> 61);
    best.seq = bk & ((1ull << 61) - 1);
    best.src = bsi >> 28;
    best.idx = bsi & ((1 << 28) - 1);
    s.algo_bytes += 16LL * na + 24LL * ne;
    return best;
  }

  MF_FN void pool_remove(int i) {
    const int last = s.n_ev - 1;
    g.sync();
    if (g.leader() && i != last) {
      I.e_t[i] = I.e_t[last];
      I.e_seq[i] = I.e_seq[last];
      I.e_kind[i] = I.e_kind[last];
      I.e_a[i] = I.e_a[last];
      I.e_b[i] = I.e_b[last];
    }
    g.sync();
    --s.n_ev;
  }

  // ----------------------------------------------------- active flow set
  MF_FN void remove_active(int fid) {  // engine.cpp:251-259
    const int pos = I.f_apos[fid];
    if (pos >= 0) remove_active_at(fid, pos);
  }
  MF_FN void remove_active_at(int fid, int pos) {
    const int last = s.n_active - 1;
    const int lf = I.a_fid[last];
    if (I.TS_cap > 0) {  // the leaving flow releases its route's slots
      int nf = s.sl_nfree, un = s.n_unslotted;
      g.sync();
      if (g.leader()) {
        const int rn = I.a_rn[pos];
        for (int k = 0; k < rn; ++k) {
          const int sl = I.a_sl[pos * I.rmax + k];
          if (sl == 0xFFFF) {
            --un;
            continue;
          }
          const int ref = I.sl_ref[sl] - 1;
          I.sl_ref[sl] = (unsigned short)ref;
          if (ref == 0) {
            I.l2s[I.sl_link[sl]] = 0xFFFFu;
            I.sl_free[nf++] = (unsigned short)sl;
          }
        }
      }
      g.sync();
      s.sl_nfree = g.shfl(nf, 0);
      s.n_unslotted = g.shfl(un, 0);
    }
    g.sync();
    if (g.leader()) {
      I.a_fid[pos] = lf;
      I.a_rem[pos] = I.a_rem[last];
      I.a_rate[pos] = I.a_rate[last];
      I.a_evt[pos] = I.a_evt[last];
      I.a_evseq[pos] = I.a_evseq[last];
      I.a_rn[pos] = I.a_rn[last];
      I.f_apos[lf] = pos;
      I.f_apos[fid] = -1;
    }
    const int rm = I.rmax;
    for (int k = g.lane(); k < rm; k += G::N) {
      I.a_rl[pos * rm + k] = I.a_rl[last * rm + k];
      I.a_sl[pos * rm + k] = I.a_sl[last * rm + k];
    }
    g.sync();
    --s.n_active;
  }

  MF_FN void advance_to(double t) {  // engine.cpp:261-276
    const double dt = dsub(t, s.now);
    if (!(dt > -1e-9)) {
      fail(ERR_INTERNAL, CHK_TIME_BACKWARDS);
      return;
    }
    if (dt > 0.0) {
      const int na = s.n_active;
      double* __restrict__ rem = I.a_rem;
      const double* __restrict__ rt = I.a_rate;
      bool bad = false;
MF_UNROLL
      for (int p = g.lane(); p < na; p += G::N) {
        double x = dsub(rem[p], dmul(rt[p], dt));
        if (x < 0.0) {
          const double sz = I.f_size[I.a_fid[p]];
          if (!(x > dsub(-dmul(1e-6, smax(sz, 1.0)), 1e-9))) bad = true;
          x = 0.0;
        }
        rem[p] = x;
      }
      g.sync();
      s.algo_bytes += 24LL * na;
      if (g.any(bad)) {
        fail(ERR_INTERNAL, CHK_OVERSHOOT);
        return;
      }
    }
    s.now = t;
  }

  // --------------------------------------------------------- pipeline info
  // per-layer scans run one layer per lane (votes), layers in order
  MF_FN int l_curr(int b) {  // engine.cpp:712-720
    const int L = I.b_layers[b];
    const int base = I.b_lbase[b];
    for (int l0 = 0; l0 < L; l0 += G::N) {
      const int l = l0 + g.lane();
      bool hit = false;
      if (l < L) {
        const int c = I.pl_coll[base + l];
        hit = !I.pl_done[base + l] || (c >= 0 && I.c_open[c] > 0);
      }
      const unsigned m = g.ballot(hit);
      if (m) return l0 + ctz32(m) + 1;
    }
    return L > 1 ? L : 1;
  }
  MF_FN double remaining_compute(int b) {  // engine.cpp:722-728, summed in layer order
    const int L = I.b_layers[b];
    const int base = I.b_lbase[b];
    double total = 0.0;
    for (int l0 = 0; l0 < L; l0 += G::N) {
      const int l = l0 + g.lane();
      double v = 0.0;
      bool use = false;
      if (l < L) {
        use = !I.pl_done[base + l];
        v = I.pl_cost[base + l];
      }
      const unsigned m = g.ballot(use);
      const int cnt = (L - l0) < G::N ? (L - l0) : G::N;
      for (int k = 0; k < cnt; ++k) {
        const double x = g.shfl(v, k);
        if (m & (1u << k)) total = dadd(total, x);
      }
    }
    return total;
  }
  MF_FN bool batch_drained(int b) const {  // engine.cpp:730-734
    return I.b_done[b] != kNoTime && I.b_open[b] == 0;
  }
  // all layers computed and every collective closed (engine.cpp:387-390)
  MF_FN bool pipeline_complete(int b) {
    const int L = I.b_layers[b];
    const int base = I.b_lbase[b];
    bool bad = false;
    for (int l = g.lane(); l < L; l += G::N) {
      const int c = I.pl_coll[base + l];
      if (!I.pl_done[base + l] || (c >= 0 && I.c_open[c] > 0)) bad = true;
    }
    return !g.any(bad);
  }

  // ========================================================= K2: RMLQ
  MF_FN int mlu_level(double v) {  // rmlq.cpp:29-34
    if (!(v >= 0.0)) {
      fail(ERR_INTERNAL, CHK_NEG_MLU);
      return I.p.K;
    }
    for (int i = 1; i <= I.p.K - 1; ++i)
      if (v >= I.p.thr[i - 1]) return i;
    return I.p.K;
  }

  // Stable bucketing of n entries (route position x_seg[e] = slot id in slot
  // mode, link id otherwise; key x_hi[e]; value x_val[e]; payload x_aux[e])
  // into y_key / y_val / y_aux: a warp counting sort whose scatter ranks equal
  // keys by lane (match_any), so each bucket keeps entry order. Slot mode uses
  // the on-chip per-slot counters; link mode the per-link arrays in HBM.
  // Query a bucket with bucket_at() / bucket_of(); bucket_release() after.
  MF_FN bool slot_mode() const { return I.TS_cap > 0 && s.n_unslotted == 0; }
  MF_FN int entry_key(int p, int k) const { return slot_mode() ? I.a_sl[p * I.rmax + k] : arl(p, k); }

  MF_FN int bucket_by_link(int n) {
    s.bk_slots = slot_mode();
    int* cntp = s.bk_slots ? I.sl_cnt : I.l_cnt;
    int* offp = s.bk_slots ? I.sl_end : I.l_off;
    unsigned short* tlp = s.bk_slots ? I.sl_tl : I.s_tl;
    if (s.bk_slots) {
      for (int j = g.lane(); j < s.sl_hw; j += G::N) I.sl_cnt[j] = 0;
      g.sync();
    }
    int nt = 0;
    for (int base = 0; base < n; base += G::N) {
      const int e = base + g.lane();
      bool first = false;
      int l = 0;
      if (e < n) {
        l = I.x_seg[e];
        first = g.atomic_add(&cntp[l], 1) == 0;
      }
      const unsigned m = g.ballot(first);
      if (first) tlp[nt + popc32(m & g.lanemask_lt())] = (unsigned short)l;
      nt += popc32(m);
    }
    g.sync();
    int off = 0;
    for (int base = 0; base < nt; base += G::N) {
      const int j = base + g.lane();
      int c = 0, l = 0;
      if (j < nt) {
        l = tlp[j];
        c = cntp[l];
      }
      int tot;
      const int o = g.excl_scan(c, &tot);
      if (j < nt) {
        offp[l] = off + o;
        if (s.bk_slots) I.sl_mb[l] = off + o;
      }
      off += tot;
    }
    g.sync();
    for (int base = 0; base < n; base += G::N) {
      const int e = base + g.lane();
      const int l = e < n ? I.x_seg[e] : -1 - g.lane();
      const unsigned peers = g.match_any(l);
      int pos = 0;
      if (e < n) {
        pos = offp[l] + popc32(peers & g.lanemask_lt());
        I.y_key[pos] = I.x_hi[e];
        I.y_val[pos] = I.x_val[e];
        I.y_aux[pos] = I.x_aux[e];
      }
      g.sync();
      if (e < n && (peers >> g.lane()) == 1u) offp[l] = pos + 1;
      g.sync();
    }
    s.bk_n = nt;
    return nt;
  }
  // j-th bucket: its link and entry range [*e0, *e1)
  MF_FN int bucket_at(int j, int* e0, int* e1) const {
    if (s.bk_slots) {
      const int sl = I.sl_tl[j];
      *e0 = I.sl_mb[sl];
      *e1 = I.sl_end[sl];
      return I.sl_link[sl];
    }
    const int l = I.s_tl[j];
    *e1 = I.l_off[l];
    *e0 = *e1 - I.l_cnt[l];
    return l;
  }
  // entry range of link l (false when l has no entries)
  MF_FN bool bucket_of(int l, int* e0, int* e1) const {
    if (s.bk_slots) {
      const int sl = I.l2s[l];
      if (sl == 0xFFFF || I.sl_cnt[sl] == 0) return false;
      *e0 = I.sl_mb[sl];
      *e1 = I.sl_end[sl];
      return true;
    }
    const int c = I.l_cnt[l];
    if (c == 0) return false;
    *e1 = I.l_off[l];
    *e0 = *e1 - c;
    return true;
  }
  MF_FN void bucket_release(int nt) {
    if (s.bk_slots) {
      for (int j = g.lane(); j < nt; j += G::N) I.sl_cnt[I.sl_tl[j]] = 0;
    } else {
      for (int j = g.lane(); j < nt; j += G::N) I.l_cnt[I.s_tl[j]] = 0;
    }
    g.sync();
  }

  // LinkLoadIndex (allocator.cpp:143-161): entries (link, band<<16|level, rate)
  // for allocated flows with rate > 0; per link sorted by (key, rate) with
  // running sums. Returns the touched-link count (see index_release).
  MF_NOINLINE int build_index() {
    int n = 0;
    for (int base = 0; base < s.n_active; base += G::N) {
      const int p = base + g.lane();
      int c = 0;
      if (p < s.n_active && I.a_rate[p] > 0.0) c = arn(p);
      int tot;
      const int off = g.excl_scan(c, &tot);
      if (c > 0) {
        const int fid = I.a_fid[p];
        const unsigned long long key = ((unsigned long long)I.f_band[fid] << 16) | I.f_level[fid];
        const double r = I.a_rate[p];
        const int hx = I.f_hidx[fid];
        for (int k = 0; k < c; ++k) {
          I.x_seg[n + off + k] = entry_key(p, k);
          I.x_hi[n + off + k] = key;
          I.x_val[n + off + k] = r;
          I.x_aux[n + off + k] = hx;
        }
      }
      n += tot;
    }
    g.sync();
    if (n > I.X_cap) {
      fail(ERR_INTERNAL, CHK_CAP_SCRATCH);
      return 0;
    }
    const int nt = bucket_by_link(n);
    // per link: insertion sort by (key, rate), then running sums in that order
    for (int j = g.lane(); j < nt; j += G::N) {
      int e0, e1;
      bucket_at(j, &e0, &e1);
      for (int a = e0 + 1; a < e1; ++a) {
        const unsigned long long k = I.y_key[a];
        const double v = I.y_val[a];
        const int ax = I.y_aux[a];
        const unsigned long long vb = dbits(v);
        int m = a;
        while (m > e0 && (I.y_key[m - 1] > k || (I.y_key[m - 1] == k && dbits(I.y_val[m - 1]) > vb))) {
          I.y_key[m] = I.y_key[m - 1];
          I.y_val[m] = I.y_val[m - 1];
          I.y_aux[m] = I.y_aux[m - 1];
          --m;
        }
        I.y_key[m] = k;
        I.y_val[m] = v;
        I.y_aux[m] = ax;
      }
      double run = 0.0;
      for (int a = e0; a < e1; ++a) {
        run = dadd(run, I.y_val[a]);
        I.x_pre[a] = run;
      }
    }
    g.sync();
    s.algo_bytes += 40LL * n;
    return nt;
  }

  // LinkLoadIndex::higher_fraction (allocator.cpp:163-171); per-lane query
  MF_FN double index_fraction(int l, int band, int level) const {
    int e0, e1;
    if (!bucket_of(l, &e0, &e1)) return 0.0;
    const unsigned long long want = ((unsigned long long)band << 16) | (unsigned long long)level;
    int lo = e0, hi = e1;  // first entry with key >= want
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (I.y_key[mid] < want) lo = mid + 1; else hi = mid;
    }
    if (lo == e0) return 0.0;
    const double v = ddiv(I.x_pre[lo - 1], I.cap[l]);
    return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
  }

  // libstdc++ iteration order of the last allocation's rate map
  MF_NOINLINE void build_hash_order() {
    const int n = s.h_n;
    if (g.leader()) {
      int head = -1;
      int bc = 1;
      int stage = 0;
      for (int i = 0; i < n; ++i) {
        if (stage < kHashStages && i == kRehashAt[stage]) {
          int nbc = kBucketsAt[stage++];
          for (int b = 0; b < nbc; ++b) I.h_bkt[b] = -2;
          int p = head;
          head = -1;
          int bbegin = -1;
          while (p != -1) {
            int nx = I.h_next[p];
            int b = I.h_keys[p] % nbc;
            if (I.h_bkt[b] == -2) {
              I.h_next[p] = head;
              head = p;
              I.h_bkt[b] = -1;
              if (I.h_next[p] != -1) I.h_bkt[bbegin] = p;
              bbegin = b;
            } else {
              int a = I.h_bkt[b];
              if (a == -1) {
                I.h_next[p] = head;
                head = p;
              } else {
                I.h_next[p] = I.h_next[a];
                I.h_next[a] = p;
              }
            }
            p = nx;
          }
          bc = nbc;
        }
        int b = I.h_keys[i] % bc;
        if (I.h_bkt[b] != -2) {
          int a = I.h_bkt[b];
          if (a == -1) {
            I.h_next[i] = head;
            head = i;
          } else {
            I.h_next[i] = I.h_next[a];
            I.h_next[a] = i;
          }
        } else {
          I.h_next[i] = head;
          head = i;
          if (I.h_next[i] != -1) I.h_bkt[I.h_keys[I.h_next[i]] % bc] = i;
          I.h_bkt[b] = -1;
        }
      }
      int rank = 0;
      for (int p = head; p != -1; p = I.h_next[p]) I.h_rank[p] = rank++;
    }
    g.sync();
    s.h_ready = 1;
  }

  // load_fraction over a live LinkLoadIndex: the contributors of link l are
  // the bucket prefix with key < (band, level); summed in unordered_map order
  // (two or fewer: any order is exact)
  MF_NOINLINE double load_fraction_idx(int l, int band, int level) {
    int e0, e1;
    double used = 0.0;
    if (bucket_of(l, &e0, &e1)) {
      const unsigned long long want = ((unsigned long long)band << 16) | (unsigned long long)level;
      int lo = e0, hi = e1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (I.y_key[mid] < want) lo = mid + 1; else hi = mid;
      }
      const int cnt = lo - e0;
      if (cnt <= 2) {
        for (int i = e0; i < lo; ++i) used = dadd(used, I.y_val[i]);
      } else {
        if (!s.h_ready) build_hash_order();
        for (int i = g.lane(); i < cnt; i += G::N) {
          I.x_hi[i] = (unsigned long long)I.h_rank[I.y_aux[e0 + i]];
          I.x_lo[i] = 0;
          I.x_val[i] = I.y_val[e0 + i];
        }
        g.sync();
        sort_x(cnt);
        for (int i = 0; i < cnt; ++i) used = dadd(used, I.x_val[i]);
      }
    }
    const double v = ddiv(used, I.cap[l]);
    return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
  }

  // load_fraction (allocator.cpp:128-141): sum in unordered_map order
  MF_NOINLINE double load_fraction(int l, int band, int level) {
    int cnt = 0;
    for (int base = 0; base < s.n_active; base += G::N) {
      int p = base + g.lane();
      int c = 0;
      if (p < s.n_active && I.a_rate[p] > 0.0) {
        int fid = I.a_fid[p];
        if (outranks(I.f_band[fid], I.f_level[fid], band, level)) {
          const int rn = arn(p);
          for (int k = 0; k < rn; ++k)
            if (arl(p, k) == l) {
              c = 1;
              break;
            }
        }
      }
      int tot;
      int off = g.excl_scan(c, &tot);
      if (c) {
        int fid = I.a_fid[p];
        I.x_hi[cnt + off] = (unsigned long long)I.f_hidx[fid];
        I.x_lo[cnt + off] = 0;
        I.x_val[cnt + off] = I.a_rate[p];
      }
      cnt += tot;
    }
    g.sync();
    s.algo_bytes += 24LL * s.n_active;
    double used = 0.0;
    if (cnt <= 2) {
      for (int i = 0; i < cnt; ++i) used = dadd(used, I.x_val[i]);
    } else {
      if (!s.h_ready) build_hash_order();
      for (int i = g.lane(); i < cnt; i += G::N)
        I.x_hi[i] = (unsigned long long)I.h_rank[(int)I.x_hi[i]];
      g.sync();
      sort_x(cnt);
      for (int i = 0; i < cnt; ++i) used = dadd(used, I.x_val[i]);
    }
    double v = ddiv(used, I.cap[l]);
    return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
  }

  // natural_key (rmlq.cpp:101-127) -> (band, level); per-lane when idx given
  MF_FN void natural_key(int fid, int lcur, int nx, bool use_idx, int* ob, int* ol) {
    const int st = I.f_stage[fid];
    if (st != ST_P2D) {
      int v = I.f_tl[fid] - lcur;
      if (v < 0) v = 0;
      if (v > I.p.K - 1) v = I.p.K - 1;
      *ob = BD_EARLY;
      *ol = v + 1;
      return;
    }
    int pb = I.f_band[fid], pl = I.f_level[fid];
    if (pb == BD_EARLY) {
      pb = BD_DEFERRED;
      pl = I.p.K;
    }
    // compute_mlu (rmlq.cpp:43-82)
    const double size_rem = remaining(fid);
    const double time_rem = dsub(I.f_dl[fid], s.now);
    const int rn = rlen(fid), rb = rbeg(fid);
    double value;
    if (rn == 0) {
      value = 0.0;
    } else {
      double best_eff = MF_INF;
      for (int k = 0; k < rn; ++k) {
        int l = I.route_links[rb + k];
        double rho = use_idx ? index_fraction(l, pb, pl)
                             : (s.rel_idx ? load_fraction_idx(l, pb, pl) : load_fraction(l, pb, pl));
        double eff = dmul(I.cap[l], dsub(1.0, rho));
        if (eff < best_eff) best_eff = eff;
      }
      if (size_rem <= 0.0)
        value = 0.0;
      else if (time_rem <= 0.0)
        value = MF_INF;
      else if (best_eff <= 0.0)
        value = MF_INF;
      else
        value = ddiv(size_rem, dmul(time_rem, best_eff));
    }
    int lv;
    if (!(value >= 0.0)) {
      lv = I.p.K;  // flagged below by the caller's check
      *ol = -1;
      *ob = BD_DEFERRED;
      return;
    }
    lv = I.p.K;
    for (int i = 1; i <= I.p.K - 1; ++i)
      if (value >= I.p.thr[i - 1]) {
        lv = i;
        break;
      }
    *ol = lv;
    *ob = lv == 1 ? BD_URGENT : BD_DEFERRED;
  }

  MF_FN int rank_of(int fid) const {  // rmlq.cpp:89-99
    int r = I.f_req[fid];
    if (r >= 0 && I.r_rank[r] >= 0) return I.r_rank[r];
    int b = I.f_batch[fid];
    if (b >= 0 && I.b_rank[b] >= 0) return I.b_rank[b];
    return 0;
  }

  MF_FN void on_flow_released(int fid) {  // rmlq.cpp:137-148
    if (I.p.policy != POL_MFS) return;
    const int r = I.f_req[fid];
    if (r >= 0 && I.r_pruned[r]) {
      g.sync();
      if (g.leader()) {
        I.f_band[fid] = BD_SCAV;
        I.f_level[fid] = (uint8_t)I.p.K;
      }
      g.sync();
      return;
    }
    const int b = I.f_batch[fid];
    const int lcur = b >= 0 ? l_curr(b) : 1;
    int nb, nl;
    natural_key(fid, lcur, 0, false, &nb, &nl);
    if (nl < 0) {
      fail(ERR_INTERNAL, CHK_NEG_MLU);
      return;
    }
    const int rk = rank_of(fid);
    g.sync();
    if (g.leader()) {
      I.f_band[fid] = (uint8_t)nb;
      I.f_level[fid] = (uint8_t)nl;
      I.f_rank[fid] = rk;
    }
    g.sync();
    if (nb == BD_URGENT && I.f_stage[fid] != ST_P2D) fail(ERR_INTERNAL, CHK_URGENT_BAND);
  }

  // promote over a batch (rmlq.cpp:150-193); p2d_only for the periodic tick
  MF_NOINLINE bool promote_batch(int b, bool p2d_only) {
    MF_TIC(tp);
    const int nx = build_index();
    if (s.err) return false;
    const int lcur = l_curr(b);
    const int f0 = I.b_ffirst[b], fc = I.b_fcount[b];
    bool changed = false, bad = false, urgent_bad = false;
    for (int i = g.lane(); i < fc; i += G::N) {
      const int fid = f0 + i;
      const int stt = I.f_state[fid];
      if (stt == FL_DONE || stt == FL_PRUNED) continue;
      if (p2d_only && I.f_stage[fid] != ST_P2D) continue;
      if (I.f_band[fid] == BD_SCAV) continue;
      int nb, nl;
      natural_key(fid, lcur, nx, true, &nb, &nl);
      if (nl < 0) {
        bad = true;
        continue;
      }
      if (!outranks(nb, nl, I.f_band[fid], I.f_level[fid])) continue;
      I.f_band[fid] = (uint8_t)nb;
      I.f_level[fid] = (uint8_t)nl;
      if (nb == BD_URGENT && I.f_stage[fid] != ST_P2D) urgent_bad = true;
      changed = true;
    }
    g.sync();
    bucket_release(nx);
    MF_TOC(OUT_CY_PROMOTE, tp);
    s.algo_bytes += 40LL * fc;
    if (g.any(bad)) fail(ERR_INTERNAL, CHK_NEG_MLU);
    if (g.any(urgent_bad)) fail(ERR_INTERNAL, CHK_URGENT_BAND);
    return g.any(changed);
  }

  MF_FN void on_layer_boundary(int b) {
    if (I.p.policy != POL_MFS) return;
    promote_batch(b, false);
  }

  // ==================================================== sorting (warp bitonic)
  MF_FN bool pos_less(int pa, int pb) const {
    if (pb < 0) return pa >= 0;
    if (pa < 0) return false;
    if (I.s_k0[pa] != I.s_k0[pb]) return I.s_k0[pa] < I.s_k0[pb];
    if (I.s_k1[pa] != I.s_k1[pb]) return I.s_k1[pa] < I.s_k1[pb];
    if (I.s_k2[pa] != I.s_k2[pb]) return I.s_k2[pa] < I.s_k2[pb];
    if (I.s_k3[pa] != I.s_k3[pb]) return I.s_k3[pa] < I.s_k3[pb];
    return I.a_fid[pa] < I.a_fid[pb];
  }
  MF_FN bool pos_same_class(int pa, int pb) const {
    return I.s_k0[pa] == I.s_k0[pb] && I.s_k1[pa] == I.s_k1[pb] && I.s_k2[pa] == I.s_k2[pb] &&
           I.s_k3[pa] == I.s_k3[pb];
  }
  MF_NOINLINE void sort_ord(int* ord, int n) {
    if (n <= 1) return;
    MF_TIC(o0);
    const int n2 = pow2ceil(n);
    for (int i = n + g.lane(); i < n2; i += G::N) ord[i] = -1;
    g.sync();
    for (int k = 2; k <= n2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = g.lane(); i < n2; i += G::N) {
          int ixj = i ^ j;
          if (ixj > i) {
            int a = ord[i], b = ord[ixj];
            bool up = (i & k) == 0;
            if (up ? pos_less(b, a) : pos_less(a, b)) {
              ord[i] = b;
              ord[ixj] = a;
            }
          }
        }
        g.sync();
      }
    }
    MF_TOC(OUT_CY_SUB + 13, o0);
  }
  // joint sort of x_hi/x_lo/x_val by (hi, lo)
  MF_FN void sort_x(int n) {
    if (n <= 1) return;
    const int n2 = pow2ceil(n);
    for (int i = n + g.lane(); i < n2; i += G::N) {
      I.x_hi[i] = ~0ull;
      I.x_lo[i] = ~0ull;
      I.x_val[i] = 0.0;
    }
    g.sync();
    for (int k = 2; k <= n2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = g.lane(); i < n2; i += G::N) {
          int ixj = i ^ j;
          if (ixj > i) {
            unsigned long long ah = I.x_hi[i], al = I.x_lo[i];
            unsigned long long bh = I.x_hi[ixj], bl = I.x_lo[ixj];
            bool b_less = bh < ah || (bh == ah && bl < al);
            bool a_less = ah < bh || (ah == bh && al < bl);
            bool up = (i & k) == 0;
            if (up ? b_less : a_less) {
              double av = I.x_val[i];
              I.x_hi[i] = bh;
              I.x_lo[i] = bl;
              I.x_val[i] = I.x_val[ixj];
              I.x_hi[ixj] = ah;
              I.x_lo[ixj] = al;
              I.x_val[ixj] = av;
            }
          }
        }
        g.sync();
      }
    }
  }

  // group s_ord[o0, o0+n) into classes of equal keys, appending to s_cls
  MF_NOINLINE int group_classes(int o0, int n, int ncls) {
    for (int base = 0; base < n; base += G::N) {
      int i = base + g.lane();
      int h = 0;
      if (i < n) h = (i == 0 || !pos_same_class(I.s_ord[o0 + i], I.s_ord[o0 + i - 1])) ? 1 : 0;
      int tot;
      int off = g.excl_scan(h, &tot);
      if (h) I.s_cls[ncls + off] = o0 + i;
      ncls += tot;
    }
    g.sync();
    return ncls;
  }

  // flow subsets of the policy orders: all active flows, those with / without a deadline
  enum { SUB_ALL = 0, SUB_DL = 1, SUB_NODL = 2 };
  MF_FN bool in_sub(int p, int mode) const {
    return mode == SUB_ALL || (has_dl(I.a_fid[p]) == (mode == SUB_DL));
  }

  // compact active positions of a subset (in active order) into ord
  MF_NOINLINE int compact(int* ord, int mode) {
    int n = 0;
    for (int base = 0; base < s.n_active; base += G::N) {
      int p = base + g.lane();
      int c = (p < s.n_active && in_sub(p, mode)) ? 1 : 0;
      int tot;
      int off = g.excl_scan(c, &tot);
      if (c) ord[n + off] = p;
      n += tot;
    }
    g.sync();
    return n;
  }

  // ================================================= K3: decide (policies)
  // Fills s_ord (class order of active positions), s_cls (class starts, with
  // sentinel) and s_cap; returns the number of classes and *has_caps.
  //
  // Sorted policies keep the previous step's order (srt, flow ids) plus the
  // flows released since (srt_add): if the surviving old order is still sorted
  // under the current keys, the new flows are merged in (O(A) per step);
  // otherwise the subset is fully re-sorted. Keys end in the flow id, so the
  // order is total and equals the reference's std::sort result either way.
  MF_NOINLINE int decide(bool* has_caps) {
    *has_caps = false;
    const int A = s.n_active;
    if (A == 0) {
      s.n_srt = 0;
      s.n_add = 0;
      return 0;
    }
    const int pol = I.p.policy;
    int ncls = 0;
    if (pol == POL_FS) {  // baselines.cpp:46-51
      for (int p = g.lane(); p < A; p += G::N) I.s_ord[p] = p;
      if (g.leader()) I.s_cls[0] = 0;
      g.sync();
      ncls = 1;
    } else if (pol == POL_SJF) {  // baselines.cpp:23-57
      for (int p = g.lane(); p < A; p += G::N) {
        I.s_k0[p] = dord(I.a_rem[p]);
        I.s_k1[p] = dord(I.f_rel[I.a_fid[p]]);
        I.s_k2[p] = 0;
        I.s_k3[p] = 0;
      }
      g.sync();
      const int n = sorted_subset(I.s_ord, SUB_ALL);
      ncls = group_classes(0, n, 0);
    } else if (pol == POL_EDF) {  // baselines.cpp:59-90
      for (int p = g.lane(); p < A; p += G::N) {
        const int fid = I.a_fid[p];
        I.s_k0[p] = dord(I.f_dl[fid]);
        I.s_k1[p] = dord(I.f_rel[fid]);
        I.s_k2[p] = 0;
        I.s_k3[p] = 0;
      }
      g.sync();
      const int ne = sorted_subset(I.s_ord, SUB_DL);
      ncls = group_classes(0, ne, 0);
      const int ni = compact(I.s_ord + ne, SUB_NODL);
      if (ni > 0) {
        if (g.leader()) I.s_cls[ncls] = ne;
        g.sync();
        ++ncls;
      }
    } else if (pol == POL_KARUNA) {  // baselines.cpp:92-135
      const int nd = compact(I.s_ord, SUB_DL);
      if (nd > 0) {
        MF_TIC(k0);
        karuna_caps(nd);
        MF_TOC(OUT_CY_SUB + 11, k0);
        if (s.err) return 0;
        *has_caps = true;
        if (g.leader()) I.s_cls[0] = 0;
        g.sync();
        ncls = 1;
      }
      for (int p = g.lane(); p < A; p += G::N) {
        I.s_k0[p] = dord(I.a_rem[p]);
        I.s_k1[p] = dord(I.f_rel[I.a_fid[p]]);
        I.s_k2[p] = 0;
        I.s_k3[p] = 0;
      }
      g.sync();
      const int nr = sorted_subset(I.s_ord + nd, SUB_NODL);
      ncls = group_classes(nd, nr, ncls);
    } else if (kAalo && pol == POL_AALO) {
      ncls = decide_aalo(A);
    } else if (kAalo && pol == POL_VARYS) {
      ncls = decide_varys(A, has_caps);
    } else {  // MFS arbitrate (rmlq.cpp:201-260)
      for (int p = g.lane(); p < A; p += G::N) {
        const int fid = I.a_fid[p];
        const int band = I.f_band[fid];
        double dl = I.f_dl[fid];
        if (isnan_(dl)) {
          const int r = I.f_req[fid];
          dl = r >= 0 ? I.r_deadline[r] : MF_INF;
        }
        double k1 = 0.0, k2 = 0.0, k3 = 0.0;
        if (band == BD_URGENT || band == BD_DEFERRED) {
          k1 = (double)I.f_level[fid];
          k2 = dl;
        } else if (band == BD_EARLY) {
          k1 = (double)I.f_level[fid];
          k2 = (double)I.f_rank[fid];
          k3 = I.f_rel[fid];
        } else {
          k1 = dl;
        }
        I.s_k0[p] = (unsigned long long)band;
        I.s_k1[p] = dord(k1);
        I.s_k2[p] = dord(k2);
        I.s_k3[p] = dord(k3);
      }
      g.sync();
      const int n = sorted_subset(I.s_ord, SUB_ALL);
      ncls = group_classes(0, n, 0);
    }
    if (g.leader()) I.s_cls[ncls] = A;
    g.sync();
    s.algo_bytes += 40LL * A;
    return ncls;
  }

  // Extension (no reference counterpart; oracle: oracle/mfsim_oracle.c decide,
  // policy 5): Aalo D-CLAS. Coflow c = (batch, target layer, stage) at
  // pl index * 3 + stage; attained a_c = pl_att[c] (finished flows' sizes, in
  // completion order) + (size - remaining) of c's active flows in active order;
  // queue = #{i < K-1 : a_c >= thr[i]}; classes by (queue, c), flows without a
  // (batch, layer) are singleton coflows after the batch coflows of their queue.
  MF_FN int aalo_coflow(int fid, int b) const {  // -1: no (batch, layer) coflow
    if (b < 0) return -1;
    const int tl = I.f_tl[fid];
    if (tl < 1 || tl > I.b_layers[b]) return -1;
    return (I.b_lbase[b] + tl - 1) * 3 + I.f_stage[fid];
  }
  MF_NOINLINE int decide_aalo(int A) {
    double* __restrict__ att = I.pl_att;
    double* __restrict__ sum = I.pl_asum;
    int* __restrict__ cx = I.x_aux;  // coflow per active position (free until the sort)
    for (int p = g.lane(); p < A; p += G::N) {
      const int fid = I.a_fid[p];
      const int b = I.f_batch[fid];
      const int c = aalo_coflow(fid, b);
      if (c >= 0) sum[c] = att[c];  // equal stores from every member
      cx[p] = c;
    }
    g.sync();
    // sequential sums in active order: per chunk of N positions, the lowest
    // lane of every coflow group adds its group's values in lane order
    for (int base = 0; base < A; base += G::N) {
      const int p = base + g.lane();
      int c = -1;
      double v = 0.0;
      if (p < A) {
        c = cx[p];
        v = dsub(I.f_size[I.a_fid[p]], I.a_rem[p]);
      }
      const unsigned grp = g.match_any(c);
      const bool lead = c >= 0 && (grp & g.lanemask_lt()) == 0u;
      double acc = lead ? sum[c] : 0.0;
      for (int k = 0; k < G::N; ++k) {
        const double vk = g.shfl(v, k);
        if (lead && ((grp >> k) & 1u)) acc = dadd(acc, vk);
      }
      if (lead) sum[c] = acc;
      g.sync();
    }
    for (int p = g.lane(); p < A; p += G::N) {
      const int fid = I.a_fid[p];
      const int c = cx[p];
      const double a = c >= 0 ? sum[c] : dsub(I.f_size[fid], I.a_rem[p]);
      int q = 0;
      while (q < I.p.K - 1 && a >= I.p.thr[q]) ++q;
      I.s_k0[p] = (unsigned long long)q;
      I.s_k1[p] = c >= 0 ? (unsigned long long)c : (1ull << 40) + (unsigned long long)fid;
      I.s_k2[p] = 0;
      I.s_k3[p] = 0;
    }
    g.sync();
    const int n = sorted_subset(I.s_ord, SUB_ALL);
    return group_classes(0, n, 0);
  }

  // Extension (no reference counterpart; oracle: oracle/mfsim_oracle.c decide,
  // policy 6): Varys-style SEBF + MADD. Coflows as in Aalo (singleton coflow
  // for a flow without a batch layer). Gamma_c = max over links of L_cl /
  // capacity, L_cl = remaining bytes of c's members routed over l summed in
  // active order; one class per coflow by (Gamma_c, coflow key); every member
  // capped at remaining / Gamma_c (uncapped for Gamma_c = 0).
  MF_NOINLINE int decide_varys(int A, bool* has_caps) {
    int* __restrict__ ord = I.x_aux;  // members grouped by coflow, active order within
    for (int p = g.lane(); p < A; p += G::N) {
      const int fid = I.a_fid[p];
      const int c = aalo_coflow(fid, I.f_batch[fid]);
      I.s_k0[p] = c >= 0 ? (unsigned long long)c : (1ull << 40) + (unsigned long long)fid;
      I.s_k1[p] = (unsigned long long)p;
      I.s_k2[p] = 0;
      I.s_k3[p] = 0;
      ord[p] = p;
    }
    double* __restrict__ L = I.l_x;  // per-link scratch, zero between coflows
    for (int p = g.lane(); p < A; p += G::N)
      for (int k = 0; k < arn(p); ++k) L[arl(p, k)] = 0.0;
    g.sync();
    sort_ord(ord, A);
    for (int g0 = 0; g0 < A;) {
      const unsigned long long key = I.s_k0[ord[g0]];
      int g1 = g0 + 1;
      for (;;) {  // end of the coflow's run
        const int i = g1 + g.lane();
        const unsigned m = g.ballot(i >= A || I.s_k0[ord[i]] != key);
        if (m) {
          g1 += ctz32(m);
          break;
        }
        g1 += G::N;
      }
      // link loads: members one after another, each over its route in parallel
      for (int i = g0; i < g1; ++i) {
        const int p = ord[i];
        const int rn = arn(p);
        const double rem = I.a_rem[p];
        for (int k = g.lane(); k < rn; k += G::N) {
          const int l = arl(p, k);
          L[l] = dadd(L[l], rem);
        }
        g.sync();
      }
      double gm = 0.0;
      for (int i = g0 + g.lane(); i < g1; i += G::N) {
        const int p = ord[i];
        const int rn = arn(p);
        for (int k = 0; k < rn; ++k) {
          const int l = arl(p, k);
          gm = smax(gm, ddiv(L[l], I.cap[l]));
        }
      }
      for (int m = G::N / 2; m > 0; m >>= 1) gm = smax(gm, g.shfl_xor(gm, m));
      g.sync();
      for (int i = g0 + g.lane(); i < g1; i += G::N) {
        const int p = ord[i];
        const int rn = arn(p);
        for (int k = 0; k < rn; ++k) L[arl(p, k)] = 0.0;
        I.s_cap[p] = gm;  // stash Gamma_c
      }
      g.sync();
      g0 = g1;
    }
    for (int p = g.lane(); p < A; p += G::N) {
      const int fid = I.a_fid[p];
      const int c = aalo_coflow(fid, I.f_batch[fid]);
      const double gam = I.s_cap[p];
      I.s_k0[p] = 0;
      I.s_k1[p] = dord(gam);
      I.s_k2[p] = c >= 0 ? (unsigned long long)c : (1ull << 40) + (unsigned long long)fid;
      I.s_k3[p] = 0;
      I.s_cap[p] = gam > 0.0 ? ddiv(I.a_rem[p], gam) : MF_INF;
    }
    g.sync();
    *has_caps = true;
    const int n = sorted_subset(I.s_ord, SUB_ALL);
    return group_classes(0, n, 0);
  }

  static constexpr int kMaxAdd = 64;  // merged into the previous order; more: full sort

  // Order repair of the survivors ord[0, n1) of the previous step's order:
  // while an adjacent pair is inverted (keys changed, e.g. SJF remaining
  // sizes crossing), both elements of every inverted pair leave for the add
  // list, appended after the n2 new flows at ord + n1. A displaced element is
  // always part of a pair, so a few passes leave a sorted subsequence. False if
  // the add list would exceed kMaxAdd.
  MF_NOINLINE bool repair_order(int* ord, int* pn1, int* pn2) {
    const int n1_0 = *pn1, n2 = *pn2;
    int n1 = n1_0, nr = 0;
    int* __restrict__ flg = I.x_aux;  // scratch outside the link bucketing
    int* __restrict__ rb = I.y_aux;
    for (;;) {
      bool any = false;
      for (int i = g.lane(); i < n1; i += G::N) {
        const int v = ord[i];
        const bool rm = (i > 0 && pos_less(v, ord[i - 1])) || (i + 1 < n1 && pos_less(ord[i + 1], v));
        flg[i] = rm ? 1 : 0;
        any = any || rm;
      }
      if (!g.any(any)) break;
      g.sync();
      int k = 0;
      for (int base = 0; base < n1; base += G::N) {
        const int i = base + g.lane();
        const bool in = i < n1;
        int v = 0;
        bool rm = false;
        if (in) {
          v = ord[i];
          rm = flg[i] != 0;
        }
        g.sync();  // every lane has read its entry before the in-place compaction
        const unsigned mk = g.ballot(in && !rm);
        if (in && !rm) ord[k + popc32(mk & g.lanemask_lt())] = v;
        k += popc32(mk);
        const unsigned mr = g.ballot(in && rm);
        if (in && rm) rb[nr + popc32(mr & g.lanemask_lt())] = v;
        nr += popc32(mr);
      }
      g.sync();
      n1 = k;
      if (nr + n2 > kMaxAdd) {  // give the survivors back (n1 + nr == n1_0) for a full sort
        for (int i = g.lane(); i < nr; i += G::N) ord[n1 + i] = rb[i];
        g.sync();
        return false;
      }
    }
    if (nr > 0) {  // add list = new flows, then the pulled survivors, at ord + n1
      for (int i = g.lane(); i < n2; i += G::N) rb[nr + i] = ord[n1_0 + i];
      g.sync();
      for (int i = g.lane(); i < nr + n2; i += G::N) ord[n1 + i] = rb[i];
      g.sync();
    }
    *pn1 = n1;
    *pn2 = n2 + nr;
    return true;
  }

  // Sorted list of the active positions p with in_sub(p, mode), written to ord.
  MF_NOINLINE int sorted_subset(int* ord, int mode) {
    MF_TIC(z0);
    const int n = sorted_subset_(ord, mode);
    MF_TOC(OUT_CY_SUB + 12, z0);
    return n;
  }
  MF_FN int sorted_subset_(int* ord, int mode) {
    if (s.n_add < 0) {  // add list overflowed: sort every member from scratch
      const int n = compact(ord, mode);
      sort_ord(ord, n);
      for (int i = g.lane(); i < n; i += G::N) I.srt[i] = I.a_fid[ord[i]];
      g.sync();
      s.n_srt = n;
      s.n_add = 0;
      return n;
    }
    // survivors of the previous order, in that order
    int n1 = 0;
    for (int base = 0; base < s.n_srt; base += G::N) {
      const int i = base + g.lane();
      int p = -1;
      if (i < s.n_srt) p = I.f_apos[I.srt[i]];
      const bool keep = p >= 0 && in_sub(p, mode);
      const unsigned m = g.ballot(keep);
      if (keep) ord[n1 + popc32(m & ((1u << g.lane()) - 1u))] = p;
      n1 += popc32(m);
    }
    // flows released since, still active and in the subset
    int n2 = 0;
    int* add = ord + n1;  // staged right after the survivors
    for (int base = 0; base < s.n_add; base += G::N) {
      const int i = base + g.lane();
      int p = -1;
      if (i < s.n_add) p = I.f_apos[I.srt_add[i]];
      const bool keep = p >= 0 && in_sub(p, mode);
      const unsigned m = g.ballot(keep);
      if (keep) add[n2 + popc32(m & ((1u << g.lane()) - 1u))] = p;
      n2 += popc32(m);
    }
    g.sync();
    // keys may have changed since the last step: pull every adjacent inversion
    // of the survivors into the add list; a full sort if that list grows large
    if (n2 > kMaxAdd || !repair_order(ord, &n1, &n2)) {
      const int n = n1 + n2;
      sort_ord(ord, n);
      for (int i = g.lane(); i < n; i += G::N) I.srt[i] = I.a_fid[ord[i]];
      g.sync();
      s.n_srt = n;
      s.n_add = 0;
      return n;
    }
    const int n = n1 + n2;
    add = ord + n1;
    if (n2 > 0) {
      // rank sort of the few new flows (pos_less is a strict total order)
      int* rb = I.y_aux;
      for (int a = g.lane(); a < n2; a += G::N) {
        const int v = add[a];
        int rk = 0;
        for (int b = 0; b < n2; ++b) rk += pos_less(add[b], v) ? 1 : 0;
        rb[rk] = v;
      }
      g.sync();
      for (int a = g.lane(); a < n2; a += G::N) add[a] = rb[a];
      g.sync();
      int* tmp = I.s_ul;  // scratch (free outside allocate)
      for (int i = g.lane(); i < n; i += G::N) {
        const int v = ord[i];
        int lo, hi, dst;
        if (i < n1) {  // rank among the new flows
          lo = 0;
          hi = n2;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (pos_less(add[mid], v)) lo = mid + 1; else hi = mid;
          }
          dst = i + lo;
        } else {  // rank among the survivors
          lo = 0;
          hi = n1;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (pos_less(ord[mid], v)) lo = mid + 1; else hi = mid;
          }
          dst = (i - n1) + lo;
        }
        tmp[dst] = v;
      }
      g.sync();
      for (int i = g.lane(); i < n; i += G::N) ord[i] = tmp[i];
      g.sync();
    }
    // remember this order (flow ids) for the next step
    for (int i = g.lane(); i < n; i += G::N) I.srt[i] = I.a_fid[ord[i]];
    g.sync();
    s.n_srt = n;
    s.n_add = 0;
    return n;
  }

  // Karuna caps for the deadline class s_ord[0, nd): per-link demand summed in
  // active order (baselines.cpp:102-133), via stable bucketing by link.
  MF_NOINLINE void karuna_caps(int nd) {
    const int A = s.n_active;
    double* __restrict__ dm = I.l_x;  // per-link demand
    for (int p = g.lane(); p < A; p += G::N) I.s_cap[p] = MF_INF;
    g.sync();
    // want = remaining / slack for positive slack; demand on the touched links zeroed
    for (int i = g.lane(); i < nd; i += G::N) {
      const int p = I.s_ord[i];
      const double slack = dsub(I.f_dl[I.a_fid[p]], s.now);
      if (slack > 0.0) {
        I.s_cap[p] = ddiv(I.a_rem[p], slack);  // stash: capped below
        const int rn = arn(p);
        for (int k = 0; k < rn; ++k) dm[arl(p, k)] = 0.0;
      }
    }
    g.sync();
    // per-link demand summed in deadline_ids (= active) order (baselines.cpp:112-118):
    // flows one after another, each adding to its (distinct) route links in parallel
    for (int i0 = 0; i0 < nd; i0 += G::N) {
      const int i = i0 + g.lane();
      int p = 0, rn = 0;
      double want = 0.0;
      if (i < nd) {
        p = I.s_ord[i];
        want = I.s_cap[p];
        if (want < MF_INF) rn = arn(p);
      }
      const int cnt = nd - i0 < G::N ? nd - i0 : G::N;
      for (int t = 0; t < cnt; ++t) {
        const int rt = g.shfl(rn, t);
        if (rt == 0) continue;
        const int pt = g.shfl(p, t);
        const double w = g.shfl(want, t);
        for (int k = g.lane(); k < rt; k += G::N) {
          const int l = arl(pt, k);
          dm[l] = dadd(dm[l], w);
        }
        g.sync();
      }
    }
    for (int i = g.lane(); i < nd; i += G::N) {
      const int p = I.s_ord[i];
      const double want = I.s_cap[p];
      if (!(want < MF_INF)) continue;  // no positive slack: uncapped
      double scale = 1.0;
      const int rn = arn(p);
      for (int k = 0; k < rn; ++k) {
        const int l = arl(p, k);
        const double c = I.cap[l];
        const double dmd = dm[l];
        if (dmd > c) scale = smin(scale, ddiv(c, dmd));
      }
      I.s_cap[p] = dmul(want, scale);
    }
    g.sync();
  }

  // ============================================ K3: strict-priority filling
  // allocator.cpp:28-126. Invariants outside this function: l_res == capacity
  // and l_cnt == 0 on every link. Within a multi-flow class l_cnt holds the
  // number of unfrozen members per link, maintained incrementally (members
  // freeze permanently), which equals the reference's per-round recount; the
  // rounds then touch only that class's links and its unfrozen members.
  MF_FN void allocate(int ncls, bool has_caps) {
    if (I.TS_cap > 0 && s.n_unslotted == 0) {
      if (chip)
        allocate_slots<true>(ncls, has_caps);
      else
        allocate_slots<false>(ncls, has_caps);
    } else {
      allocate_generic(ncls, has_caps);
    }
  }

  // per-member rounds over global-memory arrays (instances beyond the
  // shared-memory plan)
  MF_NOINLINE void allocate_generic(int ncls, bool has_caps) {
    const int A = s.n_active;
    const int RM = I.rmax;
    int* __restrict__ ord = I.s_ord;
    const int* __restrict__ afid = I.a_fid;
    const unsigned short* __restrict__ arlp = I.a_rl;
    const uint8_t* __restrict__ arnp = I.a_rn;
    double* __restrict__ res = I.l_res;
    int* __restrict__ cnt = I.l_cnt;
    double* __restrict__ rate = I.s_rate;
    int* __restrict__ ul = I.s_ul;
    unsigned short* __restrict__ tl = I.s_tl;
    const double* __restrict__ capv = I.cap;
    const double* __restrict__ scap = I.s_cap;
    // rate-map insertion order for the load_fraction hash emulation
    {
      int* __restrict__ hk = I.h_keys;
      int* __restrict__ hidx = I.f_hidx;
      for (int i = g.lane(); i < A; i += G::N) {
        const int fid = afid[ord[i]];
        hk[i] = fid;
        hidx[fid] = i;
      }
    }
    g.sync();
    s.h_n = A;
    s.h_ready = 0;
    long long rounds = 0, bytes = 0;
    for (int c = 0; c < ncls; ++c) {
      const int o0 = I.s_cls[c], o1 = I.s_cls[c + 1];
      const int n = o1 - o0;
      if (n == 1) {  // singleton: bottleneck residual, capped (allocator.cpp:42-59)
        const int p = ord[o0];
        const int rn = arnp[p];
        double r = MF_INF;
        if (has_caps) {
          const double cp = scap[p];
          if (cp < MF_INF) r = smax(0.0, cp);
        }
        double mine = MF_INF;
        for (int k = g.lane(); k < rn; k += G::N) mine = smin(mine, smax(0.0, res[arlp[p * RM + k]]));
        mine = g.min_nonneg(mine);  // smax(0, residual) >= 0
        r = smin(r, mine);
        g.sync();
        for (int k = g.lane(); k < rn; k += G::N) {
          const int l = arlp[p * RM + k];
          res[l] = dsub(res[l], r);
        }
        if (g.leader()) rate[p] = r;
        g.sync();
        bytes += 20LL * rn + 12;
        continue;
      }
      // multi-flow class: members start unfrozen at rate 0; count per link
      int nt = 0;
      for (int base = 0; base < n; base += G::N) {
        const int i = base + g.lane();
        int p = 0, rn = 0;
        if (i < n) {
          p = ord[o0 + i];
          rn = arnp[p];
          rate[p] = 0.0;
          ul[i] = p;
        }
        for (int k = 0; k < RM; ++k) {
          bool first = false;
          int l = 0;
          if (k < rn) {
            l = arlp[p * RM + k];
            first = g.atomic_add(&cnt[l], 1) == 0;
          }
          const unsigned m = g.ballot(first);
          if (first) tl[nt + popc32(m & g.lanemask_lt())] = (unsigned short)l;
          nt += popc32(m);
        }
      }
      g.sync();
      int nu = n;
      while (nu > 0) {
        ++rounds;
        // inc = min over touched links of max(0, residual) / count and cap gaps.
        // The exact quotients are only needed near the minimum: res * (1/cnt)
        // is within 2 ulp of the correctly rounded res / cnt, so every link
        // whose exact quotient can be the minimum lies within that margin of
        // the approximate minimum; only those are divided exactly.
        // lane-best share with its (residual, count) and the runner-up of a
        // different pair, as in allocate_slots
        double lmin = MF_INF, b2 = MF_INF, r1 = 0.0;
        int c1 = 1;
MF_UNROLL
        for (int j = g.lane(); j < nt; j += G::N) {
          const int l = tl[j];
          const int cn = cnt[l];
          const double r = res[l];
          if (cn > 0) {
            const double rr = smax(0.0, r);
            const double a = dmul(rr, recip(cn));
            const bool other = !(rr == r1 && cn == c1);
            if (a < lmin) {
              if (other) b2 = lmin;
              lmin = a;
              r1 = rr;
              c1 = cn;
            } else if (other) {
              b2 = smin(b2, a);
            }
          }
        }
        double cmin = MF_INF;
        if (has_caps) {
MF_UNROLL
          for (int i = g.lane(); i < nu; i += G::N) {
            const int p = ul[i];
            const double cp = scap[p];
            if (cp < MF_INF) cmin = smin(cmin, dsub(smax(0.0, cp), rate[p]));
          }
        }
        const double amin = g.min_nonneg(lmin);
        for (int m = G::N / 2; m > 0; m >>= 1) cmin = smin(cmin, g.shfl_xor(cmin, m));
        const double athr = dadd(amin, dmul(amin, 0x1p-44));
        double inc = cmin;
        // a link share may be the minimum (allocator.cpp:88-93 takes min(q, cap gap)):
        // exact quotients whenever the exact minimum can lie at or below cmin,
        // i.e. within the approximation margin of amin
        if (dsub(amin, dmul(amin, 0x1p-44)) <= cmin) {
          double q = MF_INF;
          if (g.any(b2 <= athr)) {
MF_UNROLL
            for (int j = g.lane(); j < nt; j += G::N) {
              const int l = tl[j];
              const int cn = cnt[l];
              const double r = smax(0.0, res[l]);
              if (cn > 0 && dmul(r, recip(cn)) <= athr) q = smin(q, ddiv(r, (double)cn));
            }
          } else if (lmin <= athr) {
            q = ddiv(r1, (double)c1);
          }
          inc = smin(inc, g.min_nonneg(q));  // as in allocate_slots
        }
        inc = smax(inc, 0.0);
MF_UNROLL
        for (int i = g.lane(); i < nu; i += G::N) {
          const int p = ul[i];
          rate[p] = dadd(rate[p], inc);
        }
MF_UNROLL
        for (int j = g.lane(); j < nt; j += G::N) {
          const int l = tl[j];
          const int cn = cnt[l];
          if (cn > 0) res[l] = dsub(res[l], dmul(inc, (double)cn));
        }
        g.sync();
        // freeze at the cap or on a saturated link; compact the unfrozen list
        int keep_n = 0;
        bool froze = false;
        for (int base = 0; base < nu; base += G::N) {
          const int i = base + g.lane();
          bool keep = false;
          int p = 0;
          if (i < nu) {
            p = ul[i];
            double cp = MF_INF;
            if (has_caps) {
              const double c0 = scap[p];
              if (c0 < MF_INF) cp = smax(0.0, c0);
            }
            const double cap_eps = dmul(1e-12, smax(1.0, cp == MF_INF ? 0.0 : cp));
            bool stop = rate[p] >= dsub(cp, cap_eps);
            const int rn = arnp[p];
            for (int k = 0; k < rn; ++k) {
              const int l = arlp[p * RM + k];
              const double rl = res[l];
              if (rl <= s.sat_max && rl <= dmul(1e-12, capv[l])) stop = true;
            }
            keep = !stop;
            if (stop)  // a frozen member leaves every link count for good
              for (int k = 0; k < rn; ++k) g.atomic_add(&cnt[arlp[p * RM + k]], -1);
          }
          g.sync();  // every lane has read its entry before the in-place compaction
          const unsigned m = g.ballot(keep);
          if (keep) ul[keep_n + popc32(m & g.lanemask_lt())] = p;
          keep_n += popc32(m);
          if (i < nu && !keep) froze = true;
        }
        g.sync();
        bytes += (long long)nu * (20LL * RM + 29) + 32LL * nt;
        if (!g.any(froze)) {
          fail(ERR_INTERNAL, CHK_NO_PROGRESS);
          return;
        }
        nu = keep_n;
      }
    }
    // restore l_res == capacity on every link a route of this step touched
    for (int p = g.lane(); p < A; p += G::N) {
      const int rn = arnp[p];
      for (int k = 0; k < rn; ++k) {
        const int l = arlp[p * RM + k];
        res[l] = capv[l];
      }
    }
    g.sync();
    s.classes += ncls;
    s.rounds += rounds;
    s.algo_bytes += bytes;
  }

  // class filling with the shared class rate over the link slots
  // cnt[slot] += v over one member's route slots (an ILP variant that loads
  // all slot ids before the atomics measured 3 % slower: code size)
  MF_FN void route_slots_add(int* __restrict__ cnt, const unsigned short* __restrict__ sl, int rn, int v) const {
    for (int k = 0; k < rn; ++k) g.atomic_add(&cnt[sl[k]], v);
  }

  template <bool kLinksOnChip>
  MF_NOINLINE void allocate_slots(int ncls, bool has_caps) {
    const int A = s.n_active;
    const int RM = I.rmax;
    const int hw = s.sl_hw;
    int* __restrict__ ord = I.s_ord;
    const int* __restrict__ afid = I.a_fid;
    const unsigned short* __restrict__ asl = I.a_sl;
    const uint8_t* __restrict__ arnp = I.a_rn;
    double* __restrict__ res = I.sl_res;
    int* __restrict__ cnt = I.sl_cnt;
    int* __restrict__ mb = I.sl_mb;
    int* __restrict__ mend = I.sl_end;
    unsigned short* __restrict__ tl = I.sl_tl;
    unsigned short* __restrict__ sat = I.sl_sat;
    double* __restrict__ rate = I.s_rate;
    const double* __restrict__ capv = I.cap;
    const unsigned short* __restrict__ slink = I.sl_link;
    const double* __restrict__ scap = I.s_cap;
    unsigned short* __restrict__ mem = I.c_mem;
    unsigned* __restrict__ frz = I.c_frz;  // member frozen bits, by active position
    if (kLinksOnChip) {
      MF_SH(res);
      MF_SH(cnt);
      MF_SH(mb);
      MF_SH(mend);
      MF_SH(tl);
      MF_SH(sat);
      MF_SH(frz);
    }
    MF_TIC(q0);
    if (I.p.policy == POL_MFS) {  // rate-map insertion order (load_fraction)
      int* __restrict__ hk = I.h_keys;
      int* __restrict__ hidx = I.f_hidx;
      for (int i = g.lane(); i < A; i += G::N) {
        const int fid = afid[ord[i]];
        hk[i] = fid;
        hidx[fid] = i;
      }
      s.h_n = A;
      s.h_ready = 0;
    }
    // residual = capacity on every slot (allocator.cpp:36-37), counts zero
    for (int j = g.lane(); j < hw; j += G::N) {
      res[j] = capv[slink[j]];
      cnt[j] = 0;
    }
    g.sync();
    MF_TOC(OUT_CY_SUB + 0, q0);
    long long rounds = 0, bytes = 0;
    for (int c = 0; c < ncls; ++c) {
      const int o0 = I.s_cls[c], o1 = I.s_cls[c + 1];
      const int n = o1 - o0;
      if (n == 1) {  // singleton: bottleneck residual, capped (allocator.cpp:42-59)
        const int p = ord[o0];
        const int rn = arnp[p];
        double r = MF_INF;
        if (has_caps) {
          const double cp = scap[p];
          if (cp < MF_INF) r = smax(0.0, cp);
        }
        double mine = MF_INF;
        for (int k = g.lane(); k < rn; k += G::N) mine = smin(mine, smax(0.0, res[asl[p * RM + k]]));
        mine = g.min_nonneg(mine);  // smax(0, residual) >= 0
        r = smin(r, mine);
        g.sync();
        for (int k = g.lane(); k < rn; k += G::N) {
          const int j = asl[p * RM + k];
          res[j] = dsub(res[j], r);
        }
        if (g.leader()) rate[p] = r;
        g.sync();
        bytes += 20LL * rn + 12;
        continue;
      }
      // multi-flow class (allocator.cpp:61-121). Every unfrozen member has
      // received the same sequence of increments from 0, so they share one
      // rate R; a member's rate is R at the round it freezes. Per round:
      //   inc = max(min(min_j max(0,res_j)/cnt_j, capmin - R), 0)
      //   R += inc; res_j -= inc * cnt_j on slots with unfrozen members
      //   freeze members of slots whose residual fell to <= 1e-12 * capacity
      //   and members with R >= cap - eps. capmin - R is min_p(cap_p - R)
      //   (rounding is monotone); the capped unfrozen members are one list,
      //   compacted and re-minimised by the cap pass of every round.
      MF_TIC(q1);
      int nt = 0, ncap = 0;
      double cmn = MF_INF;
      for (int w = g.lane(); w < ((A + 31) >> 5); w += G::N) frz[w] = 0u;
      for (int base = 0; base < n; base += G::N) {
        const int i = base + g.lane();
        int p = 0, rn = 0;
        bool capped = false;
        if (i < n) {
          p = ord[o0 + i];
          rn = arnp[p];
          if (has_caps) capped = scap[p] < MF_INF;
        }
        for (int k = 0; k < RM; ++k) {
          bool first = false;
          int j = 0;
          if (k < rn) {
            j = asl[p * RM + k];
            first = g.atomic_add(&cnt[j], 1) == 0;
          }
          const unsigned m = g.ballot(first);
          if (first) tl[nt + popc32(m & g.lanemask_lt())] = (unsigned short)j;
          nt += popc32(m);
        }
        const unsigned mc = g.ballot(capped);
        if (capped) {  // (cap, position) of the capped members
          const int slot = ncap + popc32(mc & g.lanemask_lt());
          const double cp = smax(0.0, scap[p]);
          I.x_hi[slot] = dbits(cp);
          I.x_lo[slot] = (unsigned long long)p;
          cmn = smin(cmn, cp);
        }
        ncap += popc32(mc);
      }
      cmn = g.min_nonneg(cmn);  // smax(0, cap) >= 0
      g.sync();
      {  // slot -> member incidence: extents from the counts, atomic fill
        int off = 0;
        for (int base = 0; base < nt; base += G::N) {
          const int jj = base + g.lane();
          int c0 = 0, j = 0;
          if (jj < nt) {
            j = tl[jj];
            c0 = cnt[j];
          }
          int tot;
          const int o = g.excl_scan(c0, &tot);
          if (jj < nt) {
            mb[j] = off + o;
            mend[j] = off + o;
          }
          off += tot;
        }
        g.sync();
        for (int i = g.lane(); i < n; i += G::N) {
          const int p = ord[o0 + i];
          const int rn = arnp[p];
          for (int k = 0; k < rn; ++k) mem[g.atomic_add(&mend[asl[p * RM + k]], 1)] = (unsigned short)p;
        }
        g.sync();
      }
      MF_TOC(OUT_CY_SUB + 1, q1);
      if (nt > s.max_touch) s.max_touch = nt;
      int nu = n;
      double R = 0.0;
      while (nu > 0) {
        ++rounds;
        MF_TIC(q2);
        const double cmin = ncap > 0 ? dsub(cmn, R) : MF_INF;
        // Approximate shares max(0,res)/cnt through a single-precision
        // reciprocal (relative error < 2^-23). Each lane keeps its best share
        // with its (residual, count) and the best share of a DIFFERENT
        // (residual, count) pair: when no lane's runner-up lies within the
        // margin of the warp minimum, the exact minimum is among the lanes'
        // best pairs and one division per lane settles it; otherwise a second
        // pass divides every share within the margin.
        double lmin = MF_INF, b2 = MF_INF, r1 = 0.0;
        int c1 = 1;
MF_UNROLL
        for (int jj = g.lane(); jj < nt; jj += G::N) {
          const int j = tl[jj];
          const int cn = cnt[j];
          const double r = res[j];
          if (cn > 0) {
            const double rr = smax(0.0, r);
            const double a = dmul(rr, frecip(cn));
            const bool other = !(rr == r1 && cn == c1);
            if (a < lmin) {
              if (other) b2 = lmin;
              lmin = a;
              r1 = rr;
              c1 = cn;
            } else if (other) {
              b2 = smin(b2, a);
            }
          }
        }
        const double amin = g.min_nonneg(lmin);  // smax(0, r) / cnt >= 0
        double inc = cmin;
        // the gate widens by the margin so that an exact minimum just below
        // cmin whose approximation rounded above it still wins (allocator.cpp:88-93)
        if (dsub(amin, dmul(amin, 0x1p-18)) <= cmin) {
          const double athr = dadd(amin, dmul(amin, 0x1p-18));
          double q = MF_INF;
          if (g.any(b2 <= athr)) {
MF_UNROLL
            for (int jj = g.lane(); jj < nt; jj += G::N) {
              const int j = tl[jj];
              const int cn = cnt[j];
              const double r = smax(0.0, res[j]);
              if (cn > 0 && dmul(r, frecip(cn)) <= athr) q = smin(q, ddiv(r, (double)cn));
            }
          } else if (lmin <= athr) {
            q = ddiv(r1, (double)c1);
          }
          // quotients are >= +0 and cmin is never -0: min{cmin, q...} is order-free
          inc = smin(inc, g.min_nonneg(q));
        }
        inc = smax(inc, 0.0);
        R = dadd(R, inc);
        MF_TOC(OUT_CY_SUB + 2, q2);
        MF_TIC(q3);
        // residual update; saturated slots collected, drained slots dropped
        int ns = 0, nt2 = 0;
        for (int base = 0; base < nt; base += G::N) {
          const int jj = base + g.lane();
          int j = 0;
          bool st = false, live = false;
          if (jj < nt) {
            j = tl[jj];
            const int cn = cnt[j];
            if (cn > 0) {
              const double r = dsub(res[j], dmul(inc, (double)cn));
              res[j] = r;
              // r <= 1e-12 * cap_j implies r <= sat_max (rounding is monotone):
              // the capacity is loaded only for the rare candidates
              st = r <= s.sat_max && r <= dmul(1e-12, capv[slink[j]]);
              live = !st;
            }
          }
          g.sync();  // all lanes read tl[jj] before the in-place compaction
          const unsigned ms = g.ballot(st);
          if (st) sat[ns + popc32(ms & g.lanemask_lt())] = (unsigned short)j;
          ns += popc32(ms);
          const unsigned ml = g.ballot(live);
          if (live) tl[nt2 + popc32(ml & g.lanemask_lt())] = (unsigned short)j;
          nt2 += popc32(ml);
        }
        g.sync();
        MF_TOC(OUT_CY_SUB + 3, q3);
        MF_TIC(q4);
        // link freezes: every unfrozen member of every saturated slot, all in
        // one pass (a member on two saturated slots is claimed once)
        int got = 0;
        for (int q = 0; q < ns; ++q) {
          const int j = sat[q];
          const int e1 = mend[j];
          for (int e = mb[j] + g.lane(); e < e1; e += G::N) {
            const int p = mem[e];
            const unsigned bit = 1u << (p & 31);
            if ((frz[p >> 5] & bit) || (g.atomic_or(&frz[p >> 5], bit) & bit)) continue;
            rate[p] = R;
            const int rn = arnp[p];
            route_slots_add(cnt, asl + p * RM, rn, -1);
            ++got;
          }
        }
        g.sync();
        // cap freezes (the same rate R, so the order against the link freezes
        // is immaterial): drop frozen entries, freeze cap - eps <= R, and take
        // the minimum cap of the survivors for the next round
        if (ncap > 0) {
          int nc2 = 0;
          double mn = MF_INF;
          for (int base = 0; base < ncap; base += G::N) {
            const int i = base + g.lane();
            bool keep = false, fz = false;
            int p = 0;
            double cp = 0.0;
            if (i < ncap) {
              p = (int)I.x_lo[i];
              if (!(frz[p >> 5] & (1u << (p & 31)))) {
                cp = bits_to_d(I.x_hi[i]);
                fz = R >= dsub(cp, dmul(1e-12, smax(1.0, cp)));
                keep = !fz;
              }
            }
            g.sync();  // every lane has read its entry before the in-place compaction
            if (fz) {
              g.atomic_or(&frz[p >> 5], 1u << (p & 31));
              rate[p] = R;
              const int rn = arnp[p];
              route_slots_add(cnt, asl + p * RM, rn, -1);
              ++got;
            }
            const unsigned mk = g.ballot(keep);
            if (keep) {
              const int slot = nc2 + popc32(mk & g.lanemask_lt());
              I.x_hi[slot] = dbits(cp);
              I.x_lo[slot] = (unsigned long long)p;
              mn = smin(mn, cp);
            }
            nc2 += popc32(mk);
          }
          mn = g.min_nonneg(mn);  // stored caps are smax(0, cap) >= 0
          g.sync();
          ncap = nc2;
          cmn = mn;
        }
        int frozen = 0;
        if (ns > 0 || has_caps) {
          int tot;
          g.excl_scan(got, &tot);
          frozen = tot;
        }
        MF_TOC(OUT_CY_SUB + 4, q4);
        bytes += 32LL * nt + 24LL * frozen;
        if (frozen == 0) {
          fail(ERR_INTERNAL, CHK_NO_PROGRESS);
          return;
        }
        nu -= frozen;
        nt = nt2;
      }
      // slot counts of this class are back to zero (every member froze)
      for (int jj = g.lane(); jj < nt; jj += G::N) cnt[tl[jj]] = 0;
      g.sync();
    }
    s.classes += ncls;
    s.rounds += rounds;
    s.algo_bytes += bytes;
  }

  // engine.cpp:278-293
  MF_NOINLINE void recompute_rates() {
    bool has_caps = false;
    MF_TIC(t0);
    int ncls = decide(&has_caps);
    MF_TOC(OUT_CY_DECIDE, t0);
    if (s.err) return;
    ++s.steps;
    MF_TIC(t1);
    allocate(ncls, has_caps);
    MF_TOC(OUT_CY_ALLOC, t1);
    if (s.err) return;
    resched();
  }

  // The rate recomputation in three parts for a lock-step gang (a barrier
  // between each): the policy classes, the filling, the completion events.
  MF_NOINLINE void settle_decide() {
    s.pend_ncls = -1;
    if (!s.dirty || s.err) return;
    bool has_caps = false;
    MF_TIC(t0);
    const int ncls = decide(&has_caps);
    MF_TOC(OUT_CY_DECIDE, t0);
    if (s.err) return;
    ++s.steps;
    s.pend_ncls = ncls;
    s.pend_caps = has_caps;
  }
  MF_NOINLINE void settle_allocate() {
    if (s.pend_ncls < 0) return;
    MF_TIC(t1);
    allocate(s.pend_ncls, s.pend_caps);
    MF_TOC(OUT_CY_ALLOC, t1);
  }
  MF_NOINLINE void settle_finish() {
    if (s.pend_ncls < 0) return;
    if (!s.err) resched();
    s.dirty = 0;
    s.pend_ncls = -1;
  }

  // changed rates -> new completion events, pushed in active_ order
  // (engine.cpp:281-291)
  MF_NOINLINE void resched() {
    MF_TIC(t2);
    const int A = s.n_active;
    const unsigned long long seq0 = s.seq;
    const double now = s.now;
    const double* __restrict__ nr = I.s_rate;
    double* __restrict__ rt = I.a_rate;
    const double* __restrict__ rem = I.a_rem;
    double* __restrict__ evt = I.a_evt;
    unsigned long long* __restrict__ evs = I.a_evseq;
    int pushed = 0;
    for (int base = 0; base < A; base += G::N) {
      const int p = base + g.lane();
      int c = 0;
      double r = 0.0;
      bool chg = false;
      if (p < A) {
        r = nr[p];
        chg = !(r == rt[p]);  // exact: unchanged rates keep their old event
        c = (chg && r > 0.0) ? 1 : 0;
      }
      const unsigned m = g.ballot(c != 0);
      if (chg) {
        rt[p] = r;
        if (r > 0.0) {
          evt[p] = dadd(now, ddiv(rem[p], r));
          evs[p] = seq0 + (unsigned long long)(pushed + popc32(m & g.lanemask_lt()));
        } else {
          evs[p] = kNoSeq;
        }
      }
      pushed += popc32(m);
    }
    g.sync();
    s.seq += (unsigned long long)pushed;
    s.pushes += pushed;
    s.algo_bytes += 32LL * A;
    MF_TOC(OUT_CY_RESCHED, t2);
  }

  // ===================================================== K1: stage DAG
  MF_FN bool layer_deps_met(int b, int layer) {  // engine.cpp:356-369
    const int base = I.b_lbase[b];
    const int idx = layer - 1;
    if (layer > 1) {
      if (!I.pl_done[base + idx - 1]) return false;
      int c = I.pl_coll[base + idx - 1];
      if (c >= 0 && I.c_open[c] > 0) return false;
    }
    const int ro = I.pl_roff[base + idx], rc = I.pl_rcnt[base + idx];
    bool blocked = false;
    for (int k = g.lane(); k < rc; k += G::N) {
      int fid = I.rpool[ro + k];
      int r = I.f_req[fid];
      if (r >= 0 && I.r_pruned[r]) continue;  // waived
      if (!done(fid)) blocked = true;
    }
    return !g.any(blocked);
  }

  MF_FN void try_start_layers(int b) {  // engine.cpp:371-382
    const int L = I.b_layers[b];
    const int base = I.b_lbase[b];
    // first layer not yet started; only it may start (one layer at a time)
    int layer = 0;
    for (int l0 = 0; l0 < L && !layer; l0 += G::N) {
      const int l = l0 + g.lane();
      const unsigned m = g.ballot(l < L && !I.pl_started[base + l]);
      if (m) layer = l0 + ctz32(m) + 1;
    }
    if (!layer || !layer_deps_met(b, layer)) return;
    const int idx = base + layer - 1;
    g.sync();
    if (g.leader()) {
      I.pl_started[idx] = 1;
      I.pl_start[idx] = s.now;
    }
    g.sync();
    push(dadd(s.now, I.pl_cost[idx]), EV_COMPUTE, b, layer);
  }

  MF_FN void check_pipeline_done(int b) {  // engine.cpp:384-393
    if (I.b_done[b] != kNoTime) return;
    if (!pipeline_complete(b)) return;
    put(&I.b_done[b], s.now);
    push(s.now, EV_DEPART, b, -1);
  }

  MF_FN void try_complete_request(int r) {  // engine.cpp:585-593
    if (I.r_ttft[r] != kNoTime) return;
    const int b = I.r_batch[r];
    if (b < 0 || I.b_done[b] == kNoTime) return;
    if (I.r_open[r] > 0) return;
    double t = I.b_done[b];
    double lf = I.r_lastfin[r];
    if (lf != kNoTime) t = smax(t, lf);
    put(&I.r_ttft[r], t);
  }

  MF_NOINLINE void finish_flow(int fid) {  // engine.cpp:318-354
    // the flow's record in one burst of independent loads
    const int st = I.f_state[fid];
    const int pos = I.f_apos[fid];
    const double size = I.f_size[fid];
    const int b = I.f_batch[fid];
    const int c = I.f_cof[fid];
    const int r = I.f_req[fid];
    const int stage = I.f_stage[fid];
    if (st == FL_DONE) {
      fail(ERR_INTERNAL, CHK_FINISHED_TWICE);
      return;
    }
    if (pos >= 0) {
      const double rem = I.a_rem[pos];
      if (!(rem <= dadd(dmul(1e-6, smax(size, 1.0)), 1e-9))) {
        fail(ERR_INTERNAL, CHK_EARLY_FINISH);
        return;
      }
    }
    // owners' counters, again in one burst
    const int bopen = b >= 0 ? I.b_open[b] : 0;
    const int copen = c >= 0 ? I.c_open[c] : 1;
    const int ropen = r >= 0 ? I.r_open[r] : 0;
    const double rlast = r >= 0 ? I.r_lastfin[r] : 0.0;
    if (!(copen > 0)) {
      fail(ERR_INTERNAL, CHK_COFLOW_BARRIER);
      return;
    }
    g.sync();
    if (g.leader()) {
      I.f_state[fid] = FL_DONE;
      I.f_fin[fid] = s.now;
      if (b >= 0) I.b_open[b] = bopen - 1;
      if (c >= 0) {
        I.c_open[c] = copen - 1;
        if (copen == 1) I.c_done[c] = s.now;
      }
      if (r >= 0) {
        I.r_open[r] = ropen - 1;
        I.r_lastfin[r] = smax(rlast, s.now);
      }
      if (kAalo && I.p.policy == POL_AALO) {  // extension: attained bytes of the coflow
        const int ac = aalo_coflow(fid, b);
        if (ac >= 0) I.pl_att[ac] = dadd(I.pl_att[ac], size);
      }
    }
    g.sync();
    if (pos >= 0) remove_active_at(fid, pos);
    s.dirty = 1;
    if (c >= 0 && copen == 1) {  // barrier: the pipeline position advances
      const int cb = I.c_batch[c];
      on_layer_boundary(cb);
      if (s.err) return;
      try_start_layers(cb);
      check_pipeline_done(cb);
    }
    if (r >= 0) {
      if (stage == ST_REUSE && b >= 0) {
        try_start_layers(b);
        check_pipeline_done(b);
      }
      try_complete_request(r);
    }
  }

  MF_NOINLINE void release_flow(int fid) {  // engine.cpp:295-316
    MF_TIC(rf);
    release_flow_(fid);
    MF_TOC(OUT_CY_SUB + 7, rf);
  }
  MF_FN void release_flow_(int fid) {
    if (I.f_state[fid] != FL_PENDING) {
      fail(ERR_INTERNAL, CHK_RELEASED_TWICE);
      return;
    }
    const int r = I.f_req[fid];
    const bool pr = r >= 0 && I.r_pruned[r];
    g.sync();
    if (g.leader()) {
      I.f_rel[fid] = s.now;
      I.f_state[fid] = pr ? FL_PRUNED : FL_ACTIVE;
    }
    g.sync();
    on_flow_released(fid);
    if (s.err) return;
    const int c = I.f_cof[fid];
    if (c >= 0 && I.c_rel[c] == kNoTime) put(&I.c_rel[c], s.now);
    if (I.f_size[fid] > 0.0 && I.f_route[fid] < 0) {
      fail(ERR_SIM, CHK_ROUTE);
      return;
    }
    if (I.f_size[fid] <= 0.0 || rlen(fid) == 0) {
      finish_flow(fid);
      return;
    }
    if (s.n_active >= I.A_cap) {
      fail(ERR_INTERNAL, CHK_CAP_ACTIVE);
      return;
    }
    const int pos = s.n_active;
    const int rb = rbeg(fid), rn = rlen(fid);
    if (rn > I.rmax) {
      fail(ERR_INTERNAL, CHK_ROUTE);
      return;
    }
    g.sync();
    if (g.leader()) {
      I.a_fid[pos] = fid;
      I.a_rem[pos] = I.f_size[fid];
      I.a_rate[pos] = 0.0;
      I.a_evt[pos] = 0.0;
      I.a_evseq[pos] = kNoSeq;
      I.a_rn[pos] = (uint8_t)rn;
      I.f_apos[fid] = pos;
    }
    for (int k = g.lane(); k < rn; k += G::N)
      I.a_rl[pos * I.rmax + k] = (unsigned short)I.route_links[rb + k];
    if (I.TS_cap > 0) {  // a slot per route link, shared by every user
      int hw = s.sl_hw, nf = s.sl_nfree, un = s.n_unslotted;
      g.sync();
      if (g.leader()) {
        for (int k = 0; k < rn; ++k) {
          const int l = I.route_links[rb + k];
          int sl = I.l2s[l];
          if (sl == 0xFFFF) {
            if (nf > 0) sl = I.sl_free[--nf];
            else if (hw < I.TS_cap) sl = hw++;
            if (sl != 0xFFFF) {
              I.l2s[l] = (unsigned short)sl;
              I.sl_link[sl] = (unsigned short)l;
              I.sl_ref[sl] = 0;
            }
          }
          if (sl != 0xFFFF) I.sl_ref[sl] = (unsigned short)(I.sl_ref[sl] + 1);
          else ++un;
          I.a_sl[pos * I.rmax + k] = (unsigned short)sl;
        }
      }
      g.sync();
      s.sl_hw = g.shfl(hw, 0);
      s.sl_nfree = g.shfl(nf, 0);
      s.n_unslotted = g.shfl(un, 0);
    }
    if (I.p.policy != POL_FS && s.n_add >= 0) {
      if (s.n_add < I.A_cap) {
        if (g.leader()) I.srt_add[s.n_add] = fid;
        ++s.n_add;
      } else {
        s.n_add = -1;  // too many to merge: rebuild the order from scratch
      }
    }
    g.sync();
    ++s.n_active;
    if (s.n_active > s.max_active) s.max_active = s.n_active;
    s.dirty = 1;
  }

  MF_NOINLINE void handle_compute_complete(int b, int layer) {  // engine.cpp:395-418
    const int idx = I.b_lbase[b] + layer - 1;
    if (!(I.pl_started[idx] && !I.pl_done[idx])) {
      fail(ERR_INTERNAL, CHK_COMPUTE_STATE);
      return;
    }
    if (!layer_deps_met(b, layer)) {
      fail(ERR_INTERNAL, CHK_LAYER_DEPS);
      return;
    }
    g.sync();
    if (g.leader()) {
      I.pl_done[idx] = 1;
      I.pl_end[idx] = s.now;
    }
    g.sync();
    on_layer_boundary(b);
    if (s.err) return;
    const int c = I.pl_coll[idx];
    if (c >= 0) {
      const int mo = I.c_moff[c], mc = I.c_mcnt[c];
      for (int k = 0; k < mc; ++k) {
        int fid = I.cpool[mo + k];
        if (!(I.f_scripted[fid] & 1) && I.f_state[fid] == FL_PENDING) release_flow(fid);
        if (s.err) return;
      }
    }
    const int po = I.pl_poff[idx], pc = I.pl_pcnt[idx];
    // MFS initial P2D priorities query the last allocation per route link; in
    // workload mode no release in this loop can finish a flow (sizes > 0,
    // distinct hosts), so one index built after the promotion review serves
    // every release of the layer
    int nxr = 0;
    if (I.p.policy == POL_MFS && I.p.workload_mode && pc > 0) {
      nxr = build_index();
      if (s.err) return;
      s.rel_idx = true;
    }
    for (int k = 0; k < pc; ++k) {
      int fid = I.ppool[po + k];
      if (!(I.f_scripted[fid] & 1) && I.f_state[fid] == FL_PENDING) release_flow(fid);
      if (s.err) return;
    }
    if (s.rel_idx) {
      s.rel_idx = false;
      bucket_release(nxr);
    }
    try_start_layers(b);
    check_pipeline_done(b);
    s.dirty = 1;
  }

  MF_FN bool p2d_left(int b) {
    const int f0 = I.b_ffirst[b], fc = I.b_fcount[b];
    bool left = false;
    for (int i = g.lane(); i < fc; i += G::N) {
      int fid = f0 + i;
      if (I.f_stage[fid] == ST_P2D && !done(fid)) left = true;
    }
    return g.any(left);
  }

  MF_NOINLINE void handle_batch_depart(int b) {  // engine.cpp:420-438
    if (I.b_departed[b]) return;
    put(&I.b_departed[b], (uint8_t)1);
    if (I.p.workload_mode) {
      put(&I.u_busy[I.b_unit[b]], (uint8_t)0);
      push(s.now, EV_ADMIT, I.b_unit[b], -1);
    }
    if (p2d_left(b) && I.p.policy == POL_MFS) push(dadd(s.now, I.p.tick), EV_TICK, b, -1);
    batch_event_hook();
    if (s.err) return;
    const int mo = I.b_moff[b], mc = I.b_mcnt[b];
    for (int k = 0; k < mc; ++k) try_complete_request(I.m_pool[mo + k]);
    s.dirty = 1;
  }

  // register one flow; ids are registration order (engine.cpp:122-137)
  MF_FN int register_flow(int req, int b, int stage, int route, double size, int tl, double dl) {
    if (s.n_flows >= I.F_cap) {
      fail(ERR_INTERNAL, CHK_CAP_FLOWS);
      return -1;
    }
    const int fid = s.n_flows++;
    if (g.leader()) {
      I.f_size[fid] = size;
      I.f_rel[fid] = kNoTime;
      I.f_fin[fid] = kNoTime;
      I.f_dl[fid] = dl;
      I.f_req[fid] = req;
      I.f_batch[fid] = b;
      I.f_cof[fid] = -1;
      I.f_route[fid] = route;
      I.f_apos[fid] = -1;
      I.f_rank[fid] = 0;
      I.f_tl[fid] = tl;
      I.f_hidx[fid] = -1;
      I.f_stage[fid] = (uint8_t)stage;
      I.f_state[fid] = FL_PENDING;
      I.f_band[fid] = BD_EARLY;
      I.f_level[fid] = 1;
      I.f_scripted[fid] = 0;
      if (req >= 0) I.r_open[req] += 1;
    }
    return fid;
  }

  MF_NOINLINE void admit_batch(int unit, int moff, int mcnt) {  // engine.cpp:455-533
    if (mcnt <= 0) {
      fail(ERR_INTERNAL, CHK_EMPTY_BATCH);
      return;
    }
    if (s.n_batches >= I.B_cap) {
      fail(ERR_INTERNAL, CHK_CAP_BATCHES);
      return;
    }
    const int b = s.n_batches++;
    const int L = I.p.layers;
    const int lbase = b * L;
    double batch_tokens = 0.0;
    for (int k = 0; k < mcnt; ++k)
      batch_tokens = dadd(batch_tokens, (double)I.r_tokens[I.m_pool[moff + k]]);
    const double cost = dadd(I.p.alpha, dmul(I.p.beta, batch_tokens));
    g.sync();
    if (g.leader()) {
      I.b_unit[b] = unit;
      I.b_layers[b] = L;
      I.b_lbase[b] = lbase;
      I.b_admit[b] = s.now;
      I.b_done[b] = kNoTime;
      I.b_departed[b] = 0;
      I.b_admitted[b] = 1;
      I.b_open[b] = 0;
      I.b_rank[b] = -1;
      I.b_ffirst[b] = s.n_flows;
      I.b_fcount[b] = 0;
      I.b_moff[b] = moff;
      I.b_mcnt[b] = mcnt;
      for (int k = 0; k < mcnt; ++k) I.r_batch[I.m_pool[moff + k]] = b;
    }
    // per-layer pipeline records
    if (s.rp_top + L * mcnt > I.RP_cap || s.pp_top + L * mcnt > I.PP_cap) {
      fail(ERR_INTERNAL, CHK_CAP_POOL);
      return;
    }
    for (int i = g.lane(); i < L; i += G::N) {
      int idx = lbase + i;
      I.pl_cost[idx] = cost;
      I.pl_started[idx] = 0;
      I.pl_done[idx] = 0;
      I.pl_start[idx] = kNoTime;
      I.pl_end[idx] = kNoTime;
      I.pl_coll[idx] = -1;
      I.pl_roff[idx] = s.rp_top + i * mcnt;
      I.pl_rcnt[idx] = 0;
      I.pl_poff[idx] = s.pp_top + i * mcnt;
      I.pl_pcnt[idx] = 0;
      if (I.p.policy == POL_AALO)
        for (int k = 0; k < 3; ++k) I.pl_att[3 * idx + k] = 0.0;
    }
    g.sync();
    s.rp_top += L * mcnt;
    s.pp_top += L * mcnt;
    const int first = s.n_flows;
    // request-owned flows (build_msflows, engine.cpp:49-89)
    const double kv = I.p.kv;
    for (int k = 0; k < mcnt; ++k) {
      const int r = I.m_pool[moff + k];
      const double tokens = (double)I.r_tokens[r];
      const int u = I.r_unit[r];
      const int lc = I.r_layers[r];
      const double reuse_bytes = dmul(dmul(I.r_reuse[r], tokens), kv);
      const double p2d_bytes = dmul(tokens, kv);
      if (reuse_bytes > 0.0 && I.r_src[r] < 0) {
        fail(ERR_WORKLOAD, CHK_REUSE_SOURCE);
        return;
      }
      const double dl = I.r_deadline[r];
      const int rr = reuse_bytes > 0.0 ? I.rt_reuse[I.r_src[r] * I.p.units + u] : -1;
      const int rp = I.rt_p2d[u];
      if (s.n_flows + 2 * lc > I.F_cap) {
        fail(ERR_INTERNAL, CHK_CAP_FLOWS);
        return;
      }
      for (int l = 1; l <= lc; ++l) {
        const int idx = lbase + l - 1;
        if (reuse_bytes > 0.0) {
          int fid = register_flow(r, b, ST_REUSE, rr, reuse_bytes, l, NAN);
          if (g.leader()) {
            int n = I.pl_rcnt[idx];
            I.rpool[I.pl_roff[idx] + n] = fid;
            I.pl_rcnt[idx] = n + 1;
          }
        }
        if (p2d_bytes > 0.0) {
          int fid = register_flow(r, b, ST_P2D, rp, p2d_bytes, l, dl);
          if (g.leader()) {
            int n = I.pl_pcnt[idx];
            I.ppool[I.pl_poff[idx] + n] = fid;
            I.pl_pcnt[idx] = n + 1;
          }
        }
      }
      g.sync();
    }
    // batch-owned collectives: all-to-all among the unit's hosts
    const double coll_bytes = dmul(batch_tokens, I.p.coll);
    const int h = I.p.hpu;
    if (coll_bytes > 0.0 && h > 1) {
      const int per = h * (h - 1);
      if (s.n_flows + L * per > I.F_cap) {
        fail(ERR_INTERNAL, CHK_CAP_FLOWS);
        return;
      }
      if (s.n_coflows + L > I.C_cap || s.cm_top + L * per > I.CM_cap) {
        fail(ERR_INTERNAL, CHK_CAP_COFLOWS);
        return;
      }
      for (int l = 1; l <= L; ++l) {
        const int c = s.n_coflows++;
        const int f0 = s.n_flows;
        for (int t = g.lane(); t < per; t += G::N) {
          int i = t / (h - 1);
          int j = t % (h - 1);
          if (j >= i) ++j;
          int fid = f0 + t;
          I.f_size[fid] = coll_bytes;
          I.f_rel[fid] = kNoTime;
          I.f_fin[fid] = kNoTime;
          I.f_dl[fid] = NAN;
          I.f_req[fid] = -1;
          I.f_batch[fid] = b;
          I.f_cof[fid] = c;
          I.f_route[fid] = I.rt_coll[(unit * h + i) * h + j];
          I.f_apos[fid] = -1;
          I.f_rank[fid] = 0;
          I.f_tl[fid] = l;
          I.f_hidx[fid] = -1;
          I.f_stage[fid] = ST_COLL;
          I.f_state[fid] = FL_PENDING;
          I.f_band[fid] = BD_EARLY;
          I.f_level[fid] = 1;
          I.f_scripted[fid] = 0;
          I.cpool[s.cm_top + t] = fid;
        }
        g.sync();
        if (g.leader()) {
          I.c_batch[c] = b;
          I.c_layer[c] = l;
          I.c_open[c] = per;
          I.c_rel[c] = kNoTime;
          I.c_done[c] = kNoTime;
          I.c_moff[c] = s.cm_top;
          I.c_mcnt[c] = per;
          I.pl_coll[lbase + l - 1] = c;
        }
        g.sync();
        s.n_flows += per;
        s.cm_top += per;
      }
    }
    const int nf = s.n_flows - first;
    g.sync();
    if (g.leader()) {
      I.b_fcount[b] = nf;
      I.b_open[b] = nf;
    }
    g.sync();
    live_append(b);
    // reuse launches at admission, in (member, layer) order
    for (int k = 0; k < mcnt; ++k) {
      const int r = I.m_pool[moff + k];
      const int lc = I.r_layers[r];
      for (int l = 1; l <= lc; ++l) {
        const int idx = lbase + l - 1;
        const int ro = I.pl_roff[idx], rc = I.pl_rcnt[idx];
        for (int q = 0; q < rc; ++q) {
          int fid = I.rpool[ro + q];
          if (I.f_req[fid] == r && I.f_state[fid] == FL_PENDING) {
            release_flow(fid);
            if (s.err) return;
          }
        }
      }
    }
    put(&I.u_busy[unit], (uint8_t)1);
    try_start_layers(b);
    check_pipeline_done(b);
    batch_event_hook();
    s.dirty = 1;
  }

  MF_FN void handle_admit_try(int unit) {  // engine.cpp:440-453
    if (I.u_busy[unit]) return;
    const int head = I.q_head[unit], tail = I.q_tail[unit];
    if (head == tail) return;
    const int qo = I.q_off[unit];
    int cnt = 0;
    long long tokens = 0;
    while (head + cnt < tail) {
      const int r = I.m_pool[qo + head + cnt];
      const long long t = I.r_tokens[r];
      if (cnt > 0 && tokens + t > I.p.max_batch_tokens) break;
      ++cnt;
      tokens += t;
    }
    put(&I.q_head[unit], head + cnt);
    admit_batch(unit, qo + head, cnt);
  }

  MF_NOINLINE void activate_manual_batch(int b) {  // engine.cpp:541-558
    if (I.b_admitted[b]) return;
    put(&I.b_admitted[b], (uint8_t)1);
    const int f0 = I.b_ffirst[b], fc = I.b_fcount[b];
    for (int i = 0; i < fc; ++i) {
      const int fid = f0 + i;
      if (I.f_scripted[fid] & 1) {
        push(smax(s.now, I.f_relat[fid]), EV_RELEASE, fid, -1);
      } else if (I.f_stage[fid] == ST_REUSE) {
        release_flow(fid);
      }
      if (s.err) return;
    }
    try_start_layers(b);
    check_pipeline_done(b);
    batch_event_hook();
    s.dirty = 1;
  }

  MF_FN void live_append(int b) {
    if (s.n_live >= I.B_cap) {
      fail(ERR_INTERNAL, CHK_CAP_BATCHES);
      return;
    }
    put(&I.g_batches[s.n_live], b);
    ++s.n_live;
  }

  // =============================================== K5: MFS Algorithm 1
  MF_NOINLINE void batch_event_hook() {  // engine.cpp:560-583
    if (I.p.policy != POL_MFS) return;
    MF_TIC(tb);
    int np = on_batch_event();
    MF_TOC(OUT_CY_BATCHEV, tb);
    if (s.err || np == 0) return;
    // apply_prunes, ascending request id
    for (int k = 0; k < np; ++k) {
      const int r = I.g_pruned[k];
      put(&I.r_pruned[r], (uint8_t)1);
      const int b = I.r_batch[r];
      if (b < 0) continue;
      const int f0 = I.b_ffirst[b], fc = I.b_fcount[b];
      for (int i = g.lane(); i < fc; i += G::N) {
        int fid = f0 + i;
        if (I.f_req[fid] != r || I.f_state[fid] == FL_DONE) continue;
        I.f_band[fid] = BD_SCAV;
        if (I.f_state[fid] == FL_ACTIVE) I.f_state[fid] = FL_PRUNED;
      }
      g.sync();
      try_start_layers(b);
      check_pipeline_done(b);
    }
    s.pruned += np;
    s.dirty = 1;
  }

  // request load on one link from its sparse vector
  MF_FN double req_load(int j, int l) const {
    const int o = I.g_loff[j], n = I.g_lcnt[j];
    for (int k = 0; k < n; ++k)
      if (I.g_link[o + k] == l) return I.g_load[o + k];
    return 0.0;
  }

  // est_finish_time (inter_request.cpp:53-78) over the dense S (l_x) + L (l_y)
  MF_FN double est_finish(double comp, int* u_star) {
    double worst = 0.0;
    int ustar = 0;
    for (int u = g.lane(); u < I.nlinks; u += G::N) {
      double total = dadd(I.l_x[u], I.l_y[u]);
      double ratio = ddiv(total, I.cap[u]);
      if (ratio > worst) {
        worst = ratio;
        ustar = u;
      }
    }
    for (int m = G::N / 2; m > 0; m >>= 1) {
      double ow = g.shfl_xor(worst, m);
      int ou = g.shfl_xor(ustar, m);
      if (ow > worst || (ow == worst && ou < ustar)) {
        worst = ow;
        ustar = ou;
      }
    }
    if (worst == 0.0) ustar = 0;
    *u_star = ustar;
    return worst == MF_INF ? MF_INF : dadd(dadd(s.now, comp), worst);
  }

  // rmlq.cpp:268-382 + inter_scheduling (inter_request.cpp:90-164).
  // Returns the number of newly pruned requests (ascending, in g_pruned).
  MF_NOINLINE int on_batch_event() {
    // live (undrained) batches, creation order; drained is permanent
    int nl = 0;
    for (int base = 0; base < s.n_live; base += G::N) {
      int i = base + g.lane();
      int b = -1, c = 0;
      if (i < s.n_live) {
        b = I.g_batches[i];
        c = batch_drained(b) ? 0 : 1;
      }
      int tot;
      int off = g.excl_scan(c, &tot);
      g.sync();
      if (c) I.g_batches[nl + off] = b;
      nl += tot;
      g.sync();
    }
    s.n_live = nl;
    // in-flight unpruned requests, batch-major (slot = live batch with any)
    int nreq = 0, nb = 0;
    for (int i = 0; i < nl; ++i) {
      const int b = I.g_batches[i];
      const int mo = I.b_moff[b], mc = I.b_mcnt[b];
      int cnt = 0;
      double toks = 0.0;
      for (int k = 0; k < mc; ++k) {  // batch_tokens in member order
        int r = I.m_pool[mo + k];
        if (!I.r_pruned[r]) toks = dadd(toks, (double)I.r_tokens[r]);
      }
      for (int base = 0; base < mc; base += G::N) {
        int k = base + g.lane();
        int c = 0, r = -1;
        if (k < mc) {
          r = I.m_pool[mo + k];
          c = I.r_pruned[r] ? 0 : 1;
        }
        int tot;
        int off = g.excl_scan(c, &tot);
        if (c) {
          I.g_req[nreq + cnt + off] = r;
          I.g_rbat[nreq + cnt + off] = nb;
          I.g_inpool[nreq + cnt + off] = 0;
        }
        cnt += tot;
      }
      g.sync();
      if (cnt > 0) {
        if (g.leader()) {
          I.g_slot_b[nb] = b;
          I.g_slot_off[nb] = nreq;
          I.g_slot_cnt[nb] = cnt;
          I.g_tok[nb] = toks;
        }
        g.sync();
        ++nb;
      }
      nreq += cnt;
    }
    if (nb == 0) return 0;
    const long long in_flight = nreq;
    // per-request sparse loads (fold order: the batch's flows in id order)
    bool overflow = false;
    for (int j = g.lane(); j < nreq; j += G::N) {
      const int r = I.g_req[j];
      const int q = I.g_rbat[j];
      const int b = I.g_slot_b[q];
      const double toks = I.g_tok[q];
      const int o = j * I.LR_cap;
      int n = 0;
      const int f0 = I.b_ffirst[b], fc = I.b_fcount[b];
      for (int i = 0; i < fc && !overflow; ++i) {
        const int fid = f0 + i;
        if (done(fid)) continue;
        const double rem = remaining(fid);
        if (rem <= 0.0) continue;
        const int rn = rlen(fid);
        if (rn == 0) continue;
        double add;
        if (I.f_stage[fid] == ST_COLL) {
          if (toks <= 0.0) continue;
          add = ddiv(dmul(rem, (double)I.r_tokens[r]), toks);
        } else if (I.f_req[fid] == r) {
          add = rem;
        } else {
          continue;
        }
        const int rb = rbeg(fid);
        for (int k = 0; k < rn; ++k) {
          const int l = I.route_links[rb + k];
          int e = 0;
          while (e < n && I.g_link[o + e] != l) ++e;
          if (e == n) {
            if (n >= I.LR_cap) {
              overflow = true;
              break;
            }
            I.g_link[o + n] = l;
            I.g_load[o + n] = 0.0;
            ++n;
          }
          I.g_load[o + e] = dadd(I.g_load[o + e], add);
        }
      }
      I.g_loff[j] = o;
      I.g_lcnt[j] = n;
    }
    g.sync();
    if (g.any(overflow)) {
      fail(ERR_INTERNAL, CHK_CAP_SCRATCH);
      return 0;
    }
    // RED score per slot (inter_request.cpp:7-43) over sorted deadlines
    for (int q = g.lane(); q < nb; q += G::N) {
      const int o = I.g_slot_off[q], n = I.g_slot_cnt[q];
      for (int k = 0; k < n; ++k) {
        double d = I.r_deadline[I.g_req[o + k]];
        int m = k;
        while (m > 0 && I.g_tmp[o + m - 1] > d) {
          I.g_tmp[o + m] = I.g_tmp[o + m - 1];
          --m;
        }
        I.g_tmp[o + m] = d;
      }
      double red, dlo;
      const double d0 = I.g_tmp[o], dn = I.g_tmp[o + n - 1];
      if (n == 1 || d0 == dn) {
        red = d0;
        dlo = d0;
      } else {
        int ks = 1;
        double best = dsub(I.g_tmp[o + 1], I.g_tmp[o]);
        for (int k = 2; k < n; ++k) {
          double gap = dsub(I.g_tmp[o + k], I.g_tmp[o + k - 1]);
          if (gap > best) {
            best = gap;
            ks = k;
          }
        }
        double f = ddiv((double)ks, (double)n);
        dlo = I.g_tmp[o + ks];
        red = dadd(dmul(f, d0), dmul(dsub(1.0, f), dlo));
      }
      I.g_red[q] = red;
      I.g_dlo[q] = dlo;
      const int b = I.g_slot_b[q];
      I.g_sig[q] = q;
      I.g_sk0[q] = dord(red);
      I.g_sk1[q] = dord(I.b_admit[b]);
      I.g_sk2[q] = (unsigned long long)b;
    }
    g.sync();
    sort_slots(nb);  // sigma: (red, admit, id)
    for (int u = g.lane(); u < I.nlinks; u += G::N) I.l_x[u] = 0.0;
    g.sync();
    const long long budget =
        I.p.prune_enable ? (long long)ceil(dmul(I.p.drop_frac, (double)in_flight)) : 0;
    const long long drop_budget = budget > 0 ? budget : 0;
    int npruned = 0;
    for (int k = 0; k < nb; ++k) {
      const int q = I.g_sig[k];
      const int b = I.g_slot_b[q];
      const int o = I.g_slot_off[q], n = I.g_slot_cnt[q];
      for (int u = g.lane(); u < I.nlinks; u += G::N) I.l_y[u] = 0.0;
      g.sync();
      for (int jj = 0; jj < n; ++jj) {  // L += r.load in request order
        const int j = o + jj;
        const int lo = I.g_loff[j], ln = I.g_lcnt[j];
        for (int e = g.lane(); e < ln; e += G::N) {
          int l = I.g_link[lo + e];
          I.l_y[l] = dadd(I.l_y[l], I.g_load[lo + e]);
        }
        if (g.leader()) {
          I.g_inpool[j] = 1;
          I.g_rpos[j] = k;
        }
        g.sync();
      }
      const double comp = remaining_compute(b);
      int ustar = 0;
      double fhat = est_finish(comp, &ustar);
      const double dlo = I.g_dlo[q];
      while (fhat > dlo && npruned < drop_budget) {
        // victim: max load on u*, ties -> lowest request id
        double vload = 0.0;
        int vj = -1, vid = 0x7fffffff;
        for (int j = g.lane(); j < nreq; j += G::N) {
          if (I.g_inpool[j] != 1) continue;
          double l = req_load(j, ustar);
          if (l <= 0.0) continue;
          int id = I.g_req[j];
          if (vj < 0 || l > vload || (l == vload && id < vid)) {
            vj = j;
            vload = l;
            vid = id;
          }
        }
        for (int m = G::N / 2; m > 0; m >>= 1) {
          double ol = g.shfl_xor(vload, m);
          int oj = g.shfl_xor(vj, m);
          int oi = g.shfl_xor(vid, m);
          if (oj >= 0 && (vj < 0 || ol > vload || (ol == vload && oi < vid))) {
            vj = oj;
            vload = ol;
            vid = oi;
          }
        }
        if (vj < 0) break;  // nobody loads the bottleneck: no progress
        put(&I.g_inpool[vj], (uint8_t)2);
        put(&I.g_pruned[npruned], vid);
        ++npruned;
        double* target = (I.g_rpos[vj] == k) ? I.l_y : I.l_x;
        const int lo = I.g_loff[vj], ln = I.g_lcnt[vj];
        for (int e = g.lane(); e < ln; e += G::N) {
          int l = I.g_link[lo + e];
          target[l] = smax(0.0, dsub(target[l], I.g_load[lo + e]));
        }
        g.sync();
        fhat = est_finish(comp, &ustar);
      }
      for (int u = g.lane(); u < I.nlinks; u += G::N) I.l_x[u] = dadd(I.l_x[u], I.l_y[u]);
      g.sync();
    }
    // ranks from sigma (rmlq.cpp:355-360): every member, pruned or not
    for (int k = 0; k < nb; ++k) {
      const int b = I.g_slot_b[I.g_sig[k]];
      const int mo = I.b_moff[b], mc = I.b_mcnt[b];
      for (int i = g.lane(); i < mc; i += G::N) I.r_rank[I.m_pool[mo + i]] = k + 1;
      if (g.leader()) I.b_rank[b] = k + 1;
      g.sync();
    }
    // rerank not-done flows of every live batch (rmlq.cpp:364-373)
    for (int i = 0; i < nl; ++i) {
      const int b = I.g_batches[i];
      const int f0 = I.b_ffirst[b], fc = I.b_fcount[b];
      for (int t = g.lane(); t < fc; t += G::N) {
        int fid = f0 + t;
        if (!done(fid)) I.f_rank[fid] = rank_of(fid);
      }
      g.sync();
    }
    if (g.leader()) {  // pruned ids ascending (inter_request.cpp:162)
      for (int a = 1; a < npruned; ++a) {
        int v = I.g_pruned[a];
        int m = a;
        while (m > 0 && I.g_pruned[m - 1] > v) {
          I.g_pruned[m] = I.g_pruned[m - 1];
          --m;
        }
        I.g_pruned[m] = v;
      }
    }
    g.sync();
    s.algo_bytes += 64LL * nreq + 16LL * I.nlinks * nb;
    return npruned;
  }

  // sort sigma slots g_sig by (g_sk0, g_sk1, g_sk2)
  MF_FN bool slot_less(int a, int b) const {
    if (b < 0) return a >= 0;
    if (a < 0) return false;
    if (I.g_sk0[a] != I.g_sk0[b]) return I.g_sk0[a] < I.g_sk0[b];
    if (I.g_sk1[a] != I.g_sk1[b]) return I.g_sk1[a] < I.g_sk1[b];
    return I.g_sk2[a] < I.g_sk2[b];
  }
  MF_FN void sort_slots(int n) {
    if (n <= 1) return;
    const int n2 = pow2ceil(n);
    for (int i = n + g.lane(); i < n2; i += G::N) I.g_sig[i] = -1;
    g.sync();
    for (int k = 2; k <= n2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = g.lane(); i < n2; i += G::N) {
          int ixj = i ^ j;
          if (ixj > i) {
            int a = I.g_sig[i], b = I.g_sig[ixj];
            bool up = (i & k) == 0;
            if (up ? slot_less(b, a) : slot_less(a, b)) {
              I.g_sig[i] = b;
              I.g_sig[ixj] = a;
            }
          }
        }
        g.sync();
      }
    }
  }

  // ======================================================= main loop
  MF_FN void init_state() {
    // workload-mode state (manual mode arrives prepared by the host)
    for (int r = g.lane(); r < I.n_req; r += G::N) {
      I.r_batch[r] = -1;
      I.r_pruned[r] = 0;
      I.r_ttft[r] = kNoTime;
      I.r_open[r] = 0;
      I.r_lastfin[r] = kNoTime;
      I.r_rank[r] = -1;
    }
    for (int u = g.lane(); u < I.p.units; u += G::N) {
      I.u_busy[u] = 0;
      I.q_head[u] = 0;
      I.q_tail[u] = 0;
    }
    for (int l = g.lane(); l < I.nlinks; l += G::N) {
      I.l_res[l] = I.cap[l];
      I.l_cnt[l] = 0;
    }
    g.sync();
  }

  MF_NOINLINE void start() {
    const long long seq0 = I.seq0;
    const int n_ev0 = I.n_ev0, n_flows0 = I.n_flows0, n_batches0 = I.n_batches0,
              n_coflows0 = I.n_coflows0;
    s.now = 0.0;
    s.prev_t = -1.0;
    s.seq = (unsigned long long)seq0;
    s.events = s.steps = s.streak = s.pushes = s.algo_bytes = s.classes = s.rounds = 0;
    s.n_flows = n_flows0;
    s.n_batches = n_batches0;
    s.n_coflows = n_coflows0;
    s.n_active = 0;
    s.n_ev = n_ev0;
    s.rp_top = s.pp_top = s.cm_top = 0;
    s.next_arr = 0;
    s.epoch = 0;
    s.n_live = 0;
    s.h_n = 0;
    s.h_ready = 0;
    s.dirty = 0;
    s.err = 0;
    s.chk = 0;
    s.pruned = 0;
    s.max_active = 0;
    s.max_touch = 0;
    s.max_pool = 0;
    s.horizon = I.p.horizon;
    s.n_srt = 0;
    s.n_add = 0;
    s.sl_hw = s.sl_nfree = s.n_unslotted = 0;
    s.rel_idx = false;
    for (int k = 0; k < 32; ++k) s.cy[k] = 0;
    double cmx = 0.0;
    for (int l = g.lane(); l < I.nlinks; l += G::N) {
      I.l2s[l] = 0xFFFFu;
      cmx = smax(cmx, I.cap[l]);
    }
    for (int m = G::N / 2; m > 0; m >>= 1) cmx = smax(cmx, g.shfl_xor(cmx, m));
    s.sat_max = dmul(1e-12, cmx);
    pool_copy(true, n_ev0);  // host-prepared initial events (manual mode)
    if (!I.host_init) {
      init_state();
    } else {
      for (int l = g.lane(); l < I.nlinks; l += G::N) {
        I.l_res[l] = I.cap[l];
        I.l_cnt[l] = 0;
      }
      g.sync();
      for (int r = g.lane(); r < I.n_req; r += G::N) I.r_ttft[r] = kNoTime;
      g.sync();
      for (int b = 0; b < n_batches0; ++b) live_append(b);
    }
    recompute_rates();
    s.dirty = 0;
  }

  // pool entries between the on-chip pool and its global home
  MF_FN void pool_copy(bool to_chip, int n) {
    if (!I.e_t_home) return;
    for (int i = g.lane(); i < n; i += G::N) {
      if (to_chip) {
        I.e_t[i] = I.e_t_home[i];
        I.e_seq[i] = I.e_seq_home[i];
        I.e_kind[i] = I.e_kind_home[i];
        I.e_a[i] = I.e_a_home[i];
        I.e_b[i] = I.e_b_home[i];
      } else {
        I.e_t_home[i] = I.e_t[i];
        I.e_seq_home[i] = I.e_seq[i];
        I.e_kind_home[i] = I.e_kind[i];
        I.e_a_home[i] = I.e_a[i];
        I.e_b_home[i] = I.e_b[i];
      }
    }
    g.sync();
  }

  // Runs the instance's event loop for at most `budget` events (<= 0: to the
  // end) and, with deadline_ns, until the device clock passes it. A suspended
  // instance keeps all state in HBM plus its scalar state in sc_blob and
  // resumes exactly where it stopped. Returns true when finished. The loop is
  // begin() / step() / end() so that a gang of warps can advance their
  // instances one event at a time in lock step (engine_kernel.cu).
  MF_NOINLINE bool run(long long budget, unsigned long long deadline_ns = 0) {
    if (!begin(budget)) return false;
    int r;
    do {
      r = step(deadline_ns);
    } while (r == 0);
    return end(r == 1);
  }

  // resume or start; false when the instance finished in an earlier launch
  MF_NOINLINE bool begin(long long budget) {
    static_assert(sizeof(Sc) <= kScBlob, "scalar state exceeds its blob");
    const int ph = *I.phase;
    if (ph == 2) return false;
    if (ph == 1) {  // resume
      const unsigned int* src = reinterpret_cast<const unsigned int*>(I.sc_blob);
      unsigned int* dst = reinterpret_cast<unsigned int*>(&s);
      for (int w = 0; w < (int)(sizeof(Sc) / 4); ++w) dst[w] = src[w];
      g.sync();
      pool_copy(true, s.n_ev);
    } else {
      start();
    }
    s.stop_at = budget > 0 ? s.events + budget : 0x7fffffffffffffffLL;
    return true;
  }

  // one iteration of Engine::run's loop (engine.cpp:598-655): 0 = go on,
  // 1 = finished (or failed), 2 = suspend (event budget or deadline reached)
  MF_NOINLINE int step(unsigned long long deadline_ns) {
    const int r = step_event(deadline_ns);
    if (r == 0) settle();
    return s.err ? 1 : r;
  }
  // the rate recomputation that closes an event (engine.cpp:651-654)
  MF_NOINLINE void settle() {
    if (s.dirty && !s.err) {
      recompute_rates();
      s.dirty = 0;
    }
  }
  // the event itself: pop, advance, dispatch; leaves s.dirty for settle()
  MF_NOINLINE int step_event(unsigned long long deadline_ns) {
    const int r = step_head(deadline_ns);
    return r ? r : step_dispatch();
  }
  // pop the next event and advance the active flows to its time
  MF_NOINLINE int step_head(unsigned long long deadline_ns) {
    if (s.err) return 1;
    if (s.events >= s.stop_at) return 2;
    if (deadline_ns && now_ns() >= deadline_ns) return 2;
    MF_TIC(tn);
    Ev e = next_event();
    MF_TOC(OUT_CY_NEXT, tn);
    if (e.src == 0 || e.t > s.horizon) return 1;
    int kind, a, b;
    if (e.src == 1) {
      kind = EV_ARRIVAL;
      a = e.idx;
      b = -1;
      ++s.next_arr;
    } else if (e.src == 2) {
      kind = I.e_kind[e.idx];
      a = I.e_a[e.idx];
      b = I.e_b[e.idx];
      pool_remove(e.idx);
    } else {
      kind = EV_FLOW;
      a = I.a_fid[e.idx];
      b = -1;
    }
    MF_TIC(ta);
    advance_to(e.t);
    MF_TOC(OUT_CY_ADVANCE, ta);
    if (s.err) return 1;
#if defined(MF_TRACE) && !defined(__CUDACC__)
    fprintf(stderr, "ev %lld t=%.17g kind=%d a=%d b=%d nact=%d nev=%d\n", s.events, e.t, kind, a, b,
            s.n_active, s.n_ev);
#endif
    ++s.events;
    if (e.t == s.prev_t) {
      if (++s.streak > I.p.livelock) {
        fail(ERR_SIM, CHK_LIVELOCK);
        return 1;
      }
    } else {
      s.streak = 0;
      s.prev_t = e.t;
    }
    s.pend_kind = kind;
    s.pend_a = a;
    s.pend_b = b;
    return 0;
  }
  // the popped event's handler (engine.cpp:613-650)
  MF_NOINLINE int step_dispatch() {
    const int kind = s.pend_kind, a = s.pend_a, b = s.pend_b;
    MF_TIC(th);
    switch (kind) {
      case EV_FLOW: {
        MF_TIC(h0);
        finish_flow(a);
        MF_TOC(OUT_CY_SUB + 6, h0);
        break;
      }
      case EV_COMPUTE: {
        MF_TIC(h1);
        handle_compute_complete(a, b);
        MF_TOC(OUT_CY_SUB + 8, h1);
        break;
      }
      case EV_DEPART: {
        MF_TIC(h2);
        handle_batch_depart(a);
        MF_TOC(OUT_CY_SUB + 9, h2);
        break;
      }
      case EV_ARRIVAL: {
        const int u = I.r_unit[a];
        put(&I.q_tail[u], I.q_tail[u] + 1);
        push(s.now, EV_ADMIT, u, -1);
        break;
      }
      case EV_ADMIT: {
        MF_TIC(h3);
        if (I.p.workload_mode)
          handle_admit_try(a);
        else
          activate_manual_batch(a);
        MF_TOC(OUT_CY_SUB + 10, h3);
        break;
      }
      case EV_RELEASE:
        if (I.f_state[a] == FL_PENDING) release_flow(a);
        break;
      case EV_TICK: {
        if (p2d_left(a)) {
          if (promote_batch(a, true)) s.dirty = 1;
          push(dadd(s.now, I.p.tick), EV_TICK, a, -1);
        }
        break;
      }
      default:
        break;
    }
    MF_TOC(OUT_CY_HANDLER, th);
    return s.err ? 1 : 0;
  }

  // suspend (scalar state and pool to HBM) or finalize and publish the outputs
  MF_NOINLINE bool end(bool finished) {
    if (s.err) finished = true;
    if (!finished) {
      g.sync();
      if (g.leader()) {
        const unsigned int* src = reinterpret_cast<const unsigned int*>(&s);
        unsigned int* dst = reinterpret_cast<unsigned int*>(I.sc_blob);
        for (int w = 0; w < (int)(sizeof(Sc) / 4); ++w) dst[w] = src[w];
        *I.phase = 1;
        I.out[OUT_EVENTS] = s.events;  // progress, visible while suspended
        I.out[OUT_STEPS] = s.steps;
        I.out[OUT_ALGO_BYTES] = s.algo_bytes;
        I.out[OUT_NFLOWS] = s.n_flows;  // sizes of the partial state (a cut)
        I.out[OUT_NBATCHES] = s.n_batches;
        I.out[OUT_NCOFLOWS] = s.n_coflows;
        I.out[OUT_PRUNED] = s.pruned;
#if defined(MF_PROF)
        I.out[OUT_ROUNDS] = s.rounds;
        I.out[OUT_MAXACTIVE] = s.max_active;
        for (int k = 0; k < 32; ++k) I.out[OUT_CY_NEXT + k] = s.cy[k];
#endif
      }
      pool_copy(false, s.n_ev);
      return false;
    }
    if (!s.err) finalize();
    if (g.leader()) {
      I.out[OUT_STATUS] = s.err;
      I.out[OUT_CHECK] = s.chk;
      I.out[OUT_EVENTS] = s.events;
      I.out[OUT_STEPS] = s.steps;
      I.out[OUT_NFLOWS] = s.n_flows;
      I.out[OUT_NBATCHES] = s.n_batches;
      I.out[OUT_NCOFLOWS] = s.n_coflows;
      I.out[OUT_PRUNED] = s.pruned;
      I.out[OUT_MAXACTIVE] = s.max_active;
      I.out[OUT_PUSHES] = s.pushes;
      I.out[OUT_ALGO_BYTES] = s.algo_bytes;
      I.out[OUT_NOW_BITS] = (long long)dbits(s.now);
      I.out[OUT_CLASSES] = s.classes;
      I.out[OUT_ROUNDS] = s.rounds;
      I.out[OUT_MAXTOUCH] = s.max_touch;
      I.out[OUT_MAXPOOL] = s.max_pool;
      for (int k = 0; k < 32; ++k) I.out[OUT_CY_NEXT + k] = s.cy[k];
      *I.phase = 2;
    }
    g.sync();
    return true;
  }

  // engine.cpp:659-707: per-coflow stall and per-batch stall (coflow id order)
  MF_NOINLINE void finalize() {
    for (int c = g.lane(); c < s.n_coflows; c += G::N) {
      double stall = 0.0;
      const double dn = I.c_done[c];
      if (dn != kNoTime) {
        const int b = I.c_batch[c];
        const int layer = I.c_layer[c];
        const int base = I.b_lbase[b];
        double other = I.pl_end[base + layer - 1];
        if (layer < I.b_layers[b]) {
          const int idx = base + layer;  // reuse deps of layer + 1
          const int ro = I.pl_roff[idx], rc = I.pl_rcnt[idx];
          for (int k = 0; k < rc; ++k) {
            int fid = I.rpool[ro + k];
            int r = I.f_req[fid];
            if (r >= 0 && I.r_pruned[r]) continue;
            double fin = I.f_fin[fid];
            if (fin != kNoTime) other = smax(other, fin);
          }
        }
        stall = smax(0.0, dsub(dn, other));
      }
      I.c_stall[c] = stall;
    }
    g.sync();
    for (int b = g.lane(); b < s.n_batches; b += G::N) {
      const int L = I.b_layers[b];
      const int base = I.b_lbase[b];
      double sum = 0.0;
      int last = -1;
      for (int t = 0; t < L; ++t) {
        int nxt = 0x7fffffff;
        for (int l = 0; l < L; ++l) {
          int c = I.pl_coll[base + l];
          if (c > last && c < nxt) nxt = c;
        }
        if (nxt == 0x7fffffff) break;
        sum = dadd(sum, I.c_stall[nxt]);
        last = nxt;
      }
      I.b_stall[b] = sum;
    }
    g.sync();
    for (int r = g.lane(); r < I.n_req; r += G::N) {
      const int b = I.r_batch[r];
      I.r_stall[r] = b >= 0 ? I.b_stall[b] : 0.0;
      I.o_pruned[r] = I.r_pruned[r];
      I.o_rbatch[r] = b;
    }
    g.sync();
  }
};

}  // namespace mfb
