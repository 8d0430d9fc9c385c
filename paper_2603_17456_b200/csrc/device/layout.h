// Structure-of-arrays layout of one simulation instance in HBM.
//
// Plain C++ (no CUDA types) so the host packer (csrc/host/arena.cpp) and the
// device engine share it. Every pointer below points into one flat arena that
// the host sizes from the instance's upper bounds; the host rebases offsets to
// device addresses before upload.
//
// Reference correspondences (all under /root/reference/proj/src/core):
//   Flow (types.hpp:87-107)            -> f_* arrays, one slot per flow id
//   Engine::active_ / rate_ (engine.hpp:230-232)
//                                      -> a_* arrays in active_ order; the
//                                         completion event of an active flow
//                                         lives in its slot (a_evt/a_evseq)
//   std::priority_queue<Event> (engine.hpp:220)
//                                      -> e_* pool for non-flow events +
//                                         arrival stream + per-flow slots
//   Request / Batch / BatchPipeline / Coflow (types.hpp:117-141, engine.hpp:55-89)
//                                      -> r_*, b_*, pl_*, c_* arrays
#pragma once
#include <stdint.h>

namespace mfb {

enum : int { POL_FS = 0, POL_SJF = 1, POL_EDF = 2, POL_KARUNA = 3, POL_MFS = 4,
             POL_AALO = 5, /* extensions: no reference oracle (oracle/mfsim_oracle.c) */
             POL_VARYS = 6 };
enum : uint8_t { ST_REUSE = 0, ST_COLL = 1, ST_P2D = 2 };
enum : uint8_t { FL_PENDING = 0, FL_ACTIVE = 1, FL_DONE = 2, FL_PRUNED = 3 };
enum : uint8_t { BD_URGENT = 0, BD_EARLY = 1, BD_DEFERRED = 2, BD_SCAV = 3 };
// event kinds (engine.hpp:152-160); klass = 0 for the first three, 1 next, 2 tick
enum : uint8_t {
  EV_FLOW = 0,
  EV_COMPUTE = 1,
  EV_DEPART = 2,
  EV_ARRIVAL = 3,
  EV_ADMIT = 4,
  EV_RELEASE = 5,
  EV_TICK = 6
};

// error codes (mfsim.h:14-20) + internal check ids
enum : int {
  ERR_OK = 0,
  ERR_WORKLOAD = 3,
  ERR_SIM = 5,
  ERR_INTERNAL = 6,
};
enum : int {
  CHK_NONE = 0,
  CHK_TIME_BACKWARDS,
  CHK_OVERSHOOT,
  CHK_EARLY_FINISH,
  CHK_FINISHED_TWICE,
  CHK_RELEASED_TWICE,
  CHK_COFLOW_BARRIER,
  CHK_COMPUTE_STATE,
  CHK_LAYER_DEPS,
  CHK_NO_PROGRESS,
  CHK_URGENT_BAND,
  CHK_NEG_MLU,
  CHK_CAP_FLOWS,
  CHK_CAP_ACTIVE,
  CHK_CAP_EVENTS,
  CHK_CAP_BATCHES,
  CHK_CAP_COFLOWS,
  CHK_CAP_POOL,
  CHK_CAP_SCRATCH,
  CHK_LIVELOCK,
  CHK_EMPTY_BATCH,
  CHK_DONE_REMAINING,
  CHK_ROUTE,
  CHK_REUSE_SOURCE,
};

constexpr int kMaxK = 32;  // mfs.K upper bound on the device
constexpr int kScBlob = 1024;  // bytes reserved for the suspended scalar state

struct InstParams {
  int policy;
  int K;
  double thr[kMaxK];  // Q_1..Q_{K-1} (rmlq.cpp:8-22); aalo: Q0 * E^i
  double tick;        // EngineParams::promotion_tick
  double horizon;     // absolute
  long long livelock;
  long long max_batch_tokens;
  int layers;  // CostModel::layers (workload mode)
  double alpha, beta, kv, coll;
  int units, hpu, decode_hosts;
  int prune_enable;
  double drop_frac;
  int workload_mode;
};

struct Inst {
  InstParams p;
  // ---- sizes / capacities
  int n_req, n_arr, F_cap, B_cap, C_cap, E_cap, A_cap, PL_cap;
  int RP_cap, PP_cap, CM_cap, MP_cap, LR_cap, X_cap;
  int nlinks, rmax;  // rmax = longest route length
  int host_init;     // 1: state image prepared by the host (manual mode)
  long long seq0;    // initial push counter
  int n_ev0, n_flows0, n_batches0, n_coflows0;
  // ---- topology (shared, read-only)
  const double* cap;       // [nlinks]
  const int* route_off;    // [nroutes+1]
  const int* route_links;  // CSR
  const int* rt_reuse;     // [units*units]   lead(src) -> lead(dst)
  const int* rt_p2d;       // [units]         lead(u) -> decode(u)
  const int* rt_coll;      // [units*hpu*hpu] host(u,i) -> host(u,j)
  // ---- requests (inputs)
  const double* r_arrival;
  const double* r_deadline;
  const long long* r_tokens;
  const double* r_reuse;
  const int* r_unit;
  const int* r_src;
  const int* r_layers;
  const int* arr_order;  // request ids sorted by (arrival, id)
  const int* q_off;      // [units+1] per-unit FIFO lists
  int* m_pool;           // members: per-unit request lists (workload) / manual members
  // ---- requests (state)
  int* r_batch;
  uint8_t* r_pruned;
  double* r_ttft;  // NaN = unset
  int* r_open;
  double* r_lastfin;
  int* r_rank;  // -1 = absent from rank_ (rmlq.hpp:101)
  // ---- units
  uint8_t* u_busy;
  int* q_head;
  int* q_tail;
  // ---- flows [F_cap]
  double* f_size;
  double* f_rel;   // release_time == priority.release
  double* f_fin;   // flow_finish_, -1 = kNoTime
  double* f_dl;    // explicit deadline, NaN = none
  double* f_relat; // manual scripted release time
  int* f_req;
  int* f_batch;
  int* f_cof;
  int* f_route;
  int* f_apos;  // active_pos_
  int* f_rank;  // priority.rank
  int* f_tl;    // target_layer
  int* f_hidx;  // insertion index in the last allocation's rate map
  uint8_t* f_stage;
  uint8_t* f_state;
  uint8_t* f_band;
  uint8_t* f_level;
  uint8_t* f_scripted;
  // ---- active flows, in active_ order [A_cap]
  int* a_fid;
  double* a_rem;
  double* a_rate;
  double* a_evt;
  unsigned long long* a_evseq;  // ~0 = no pending completion event
  unsigned short* a_rl;         // route link ids, rmax per active flow
  uint8_t* a_rn;                // route length
  // ---- batches [B_cap]
  int* b_unit;
  int* b_layers;
  int* b_lbase;
  double* b_admit;
  double* b_done;  // pipeline done_t, -1 = none
  uint8_t* b_departed;
  uint8_t* b_admitted;
  int* b_open;
  int* b_rank;  // -1 = absent
  int* b_ffirst;
  int* b_fcount;
  int* b_moff;
  int* b_mcnt;
  // ---- per (batch, layer) [PL_cap]
  double* pl_cost;
  uint8_t* pl_started;
  uint8_t* pl_done;
  double* pl_start;
  double* pl_end;
  int* pl_coll;
  int* pl_roff;
  int* pl_rcnt;
  int* pl_poff;
  int* pl_pcnt;
  // aalo (extension), [3 * PL_cap] by (batch layer, stage): finished bytes, per-step sums
  double* pl_att;
  double* pl_asum;
  int* rpool;  // reuse deps  [RP_cap]
  int* ppool;  // p2d by layer [PP_cap]
  // ---- coflows [C_cap]
  int* c_batch;
  int* c_layer;
  int* c_open;
  double* c_rel;
  double* c_done;
  int* c_moff;
  int* c_mcnt;
  int* cpool;  // members [CM_cap]
  // ---- event pool [E_cap]
  double* e_t;
  unsigned long long* e_seq;
  int* e_kind;
  int* e_a;
  int* e_b;
  // ---- links [nlinks]
  double* l_res;   // == capacity outside allocate()
  int* l_cnt;      // == 0 outside a multi-flow class
  int* l_off;   // bucket cursor / end offset while entries are bucketed by link
  double* l_x;  // scratch (Karuna demand / Algorithm 1 S)
  double* l_y;  // scratch (Algorithm 1 L)
  // ---- per-step scratch [A_cap] / [X_cap = A_cap * rmax]
  double* s_rate;   // new rates by active position
  double* s_cap;    // caps by active position (+inf none)
  int* s_ord;       // class order (active positions)
  int* s_cls;       // class start offsets (+1 sentinel)
  int* s_ul;        // unfrozen members of the class being filled
  // Link slots (engine allocate_slots): every link on the route of an active
  // flow holds a compact slot while any active flow uses it (refcounted,
  // assigned at release, freed when the last user leaves). Bookkeeping lives
  // in HBM; the per-step filling state per slot is small enough for shared
  // memory. Flows that find no free slot fall back to per-link filling.
  int TS_cap;              // slot capacity (0: always the per-link variant)
  unsigned short* l2s;     // [nlinks] link -> slot, 0xFFFF = none
  unsigned short* a_sl;    // [A_cap * rmax] slot ids of active routes
  unsigned short* sl_link; // [TS] slot -> link
  unsigned short* sl_ref;  // [TS] active route entries using the slot
  unsigned short* sl_free; // [TS] free-slot stack
  double* sl_res;          // [TS] per-step residual
  int* sl_cnt;             // [TS] per-step count (unfrozen class members / bucket sizes)
  int* sl_mb;              // [TS] per-step list start
  int* sl_end;             // [TS] per-step list end / fill cursor
  unsigned short* sl_tl;   // [TS] live slots of the class
  unsigned short* sl_sat;  // [TS] slots saturated this round
  unsigned short* c_mem;   // [A_cap * rmax] slot -> member incidence
  unsigned* c_frz;         // [(A_cap+31)/32] member frozen bits
  unsigned short* s_tl;  // links touched by that class [nlinks]
  int* srt;         // sorted-subset order of the last decide (flow ids)
  int* srt_add;     // flows released since the last decide
  unsigned long long* s_k0;
  unsigned long long* s_k1;
  unsigned long long* s_k2;
  unsigned long long* s_k3;
  int* h_keys;      // last allocation's insertion sequence (flow ids)
  int* h_next;      // hash-order emulation
  int* h_bkt;
  int* h_rank;
  unsigned long long* x_hi;  // (link, key) entries [X_cap]
  unsigned long long* x_lo;
  double* x_val;
  double* x_pre;
  int* x_seg;       // segment heads / entry link ids
  unsigned long long* y_key;  // entries bucketed by link (stable)
  double* y_val;
  int* x_aux;       // per-entry payload (allocation insertion index)
  int* y_aux;
  // ---- Algorithm 1 scratch
  int* g_batches;   // live (undrained) batch list [B_cap]
  int* g_req;       // in-flight unpruned requests [n_req]
  int* g_rbat;      // sigma index of each g_req entry
  int* g_loff;      // per-request offset into g_link/g_load
  int* g_lcnt;
  int* g_link;      // [LR_cap]
  double* g_load;
  int* g_rpos;      // sigma position of each g_req entry's batch
  uint8_t* g_inpool;// 0 not yet in pool, 1 in pool, 2 pruned
  double* g_tmp;    // deadline sort scratch [n_req]
  int* g_pruned;    // newly pruned ids [n_req]
  // per slot (live batch with unpruned requests) [B_cap], sigma sort [pow2(B_cap)]
  int* g_slot_b;
  int* g_slot_off;
  int* g_slot_cnt;
  double* g_tok;
  double* g_red;
  double* g_dlo;
  int* g_sig;
  unsigned long long* g_sk0;
  unsigned long long* g_sk1;
  unsigned long long* g_sk2;
  // ---- finalize outputs
  double* c_stall;  // [C_cap]
  double* b_stall;  // [B_cap]
  double* r_stall;  // [n_req] per-request stall = its batch's stall
  uint8_t* o_pruned;  // [n_req] output copies of r_pruned / r_batch
  int* o_rbatch;
  // ---- suspend / resume across launches
  int* phase;                 // 0 fresh, 1 suspended, 2 done
  unsigned char* sc_blob;     // [kScBlob] scalar engine state while suspended
  double* e_t_home;           // global homes of an on-chip event pool (null if
  unsigned long long* e_seq_home;  //   the pool stayed in global memory)
  int* e_kind_home;
  int* e_a_home;
  int* e_b_home;
  // ---- outputs / scalars
  long long* out;  // [OUT_N]
};

enum : int {
  OUT_STATUS = 0,
  OUT_CHECK,
  OUT_EVENTS,
  OUT_STEPS,
  OUT_NFLOWS,
  OUT_NBATCHES,
  OUT_NCOFLOWS,
  OUT_PRUNED,
  OUT_MAXACTIVE,
  OUT_PUSHES,
  OUT_ALGO_BYTES,  // kernel-side algorithmic byte counter
  OUT_NOW_BITS,
  OUT_CLASSES,
  OUT_ROUNDS,
  OUT_MAXTOUCH,  // most links touched by one filled class
  OUT_MAXPOOL,   // deepest event pool
  // phase cycle counters (profiling builds, -DMF_PROF)
  OUT_CY_NEXT = 16,
  OUT_CY_ADVANCE,
  OUT_CY_HANDLER,
  OUT_CY_DECIDE,
  OUT_CY_ALLOC,
  OUT_CY_RESCHED,
  OUT_CY_BATCHEV,
  OUT_CY_PROMOTE,
  // sub-phases: allocate prep / count / inc / apply / freeze / restore,
  // finish_flow, release_flow, compute-complete, depart, admit
  OUT_CY_SUB = 24,
  OUT_N = 48
};

}  // namespace mfb
