// engine.cu -- the native SegEngine: buffers, stage sequence, timing.
//
// Mirrors SegEngine.perform_segmentation (engine.py:125-230) for a batch of
// same-sized frames: every stage is ONE launch over the whole batch, buffers
// are allocated once per engine (engine.py:110-119) and stay resident in HBM,
// and stage boundaries are CUDA events instead of perf_counter calls.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "spx_internal.cuh"

namespace spx {
int launch_convert(const uint8_t*, float*, int64_t, int64_t, int, cudaStream_t, int64_t, int64_t,
                   float);
int launch_assoc(const float*, const double*, const double*, int32_t*, const int32_t*, int64_t,
                 int64_t, int64_t, int64_t, int64_t, double, int64_t, int64_t, int, int64_t,
                 cudaStream_t);
int launch_accum_range(const float*, const int32_t*, int64_t, int64_t, double*, int64_t, int64_t,
                       int64_t, int64_t, int64_t, int64_t, int64_t, int, const int32_t*,
                       cudaStream_t);
int launch_reduce(double*, int64_t, const double*, const double*, double*, double*, int64_t*,
                  int64_t, int64_t, int64_t, int, const int32_t*, cudaStream_t);
int launch_shift(const double*, const double*, int64_t, int, double*, int32_t*, int32_t*, double,
                 cudaStream_t);
int launch_commit_done(int32_t*, int, cudaStream_t);
int launch_weak2(const int32_t*, int32_t*, int64_t, int64_t, int, cudaStream_t, int64_t, int64_t);
int launch_strict(const int32_t*, int32_t*, int64_t, int64_t, int, int64_t, int64_t, int32_t*,
                  int32_t*, int32_t*, int32_t*, cudaStream_t);
bool cell_path_ok(int64_t, int64_t, int64_t, int64_t);

namespace {

__global__ void k_gather_centres(const double* __restrict__ xy0, const double* __restrict__ lab0,
                                 const double* __restrict__ xy1, const double* __restrict__ lab1,
                                 const int32_t* __restrict__ passes, int fixed_passes, int64_t k,
                                 int frames, double* __restrict__ out_xy,
                                 double* __restrict__ out_lab, int32_t* __restrict__ out_passes) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k * frames) return;
  int64_t f = i / k;
  const int np = passes ? passes[f] : fixed_passes;
  if (out_passes && i == f * k) out_passes[f] = np;
  const bool one = np & 1;
  const double* sx = one ? xy1 : xy0;
  const double* sl = one ? lab1 : lab0;
  out_xy[2 * i] = sx[2 * i];
  out_xy[2 * i + 1] = sx[2 * i + 1];
  out_lab[3 * i] = sl[3 * i];
  out_lab[3 * i + 1] = sl[3 * i + 1];
  out_lab[3 * i + 2] = sl[3 * i + 2];
}

enum Ev { EV_START, EV_CONVERT, EV_INIT, EV_PERTURB, EV_CONN0, EV_END, EV_FIXED };


}  // namespace

struct Engine {
  spx_settings st;
  int64_t K = 0, n_bl = 0, hw = 0, max_batch = 0;
  int device = 0;
  double xy_weight = 0.0;
  float* lab = nullptr;
  int32_t* labels = nullptr;
  int32_t* scratch = nullptr;
  double* cxy[2] = {nullptr, nullptr};
  double* clab[2] = {nullptr, nullptr};
  double* slab = nullptr;
  int32_t* done = nullptr;
  int32_t* passes = nullptr;
  int32_t *cc_parent = nullptr, *cc_size = nullptr, *cc_nxt = nullptr, *cc_first = nullptr;
  ShiftTree shift_tree;  // early stop: numpy's pairwise sum of |new - old| (engine.py:196)
  CRec* rec = nullptr;   // fp32 filter records of the current centres (cell path)
  ClusterAcc* acc = nullptr;  // per-cluster update accumulators (cell path)
  int32_t* worklist = nullptr;  // flagged clusters for the exact fallback (cell path)
  int32_t* wl_n = nullptr;      // two worklist counts (pass parity), after the list
  // The exact fallback runs on a side stream, concurrently with the reduce
  // (both only need the association pass): fork / join events.
  cudaStream_t s_side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool use_cell = false;
  bool wide = false;               // S > 42: per-(cluster, strip) sums (cell.cu)
  // lanes running beside this engine, for the lanes-per-cell choice (kept
  // at 1: counting the sibling lanes measured 2-3% faster at S = 34 / 40 but
  // 12% slower for 16 VGA frames, where the doubled lanes cut latency)
  int conc = 1;
  // reduce and exact fallback as one launch (SPX_SPLIT_UPDATE=1: two
  // launches on two streams, fork / join)
  bool merged_update = !getenv("SPX_SPLIT_UPDATE");
  StripAcc* sacc = nullptr;
  long long* wwl = nullptr;
  int32_t* wwl_n = nullptr;
  cudaEvent_t ev[EV_FIXED] = {};
  std::vector<cudaEvent_t> ev_assoc, ev_update;  // start/end pairs
  int n_assoc = 0, n_update = 0;
  int64_t launches = 0;

  // ---- lanes: a large batch split into sub-batches on concurrent streams ---
  // The convert kernel is FP64-pipe bound and the association passes are
  // issue / MUFU bound, so sub-batches running concurrently overlap one
  // lane's convert (and connectivity) with another's association.  Each lane
  // is a child Engine (own buffers, worklist, side stream, events) created on
  // first use; frames are independent, so the results are bitwise the same
  // as the unsplit call (tests/test_gpu_engine.py).  Measured on C1, 256
  // frames (tools/probe.py lanes): 1 lane 4.59 ms, 2: 4.56, 3: 4.40, 4: 4.32,
  // 5: 4.67, 6: 4.48, 8: 4.44.  Staggering the lanes (lane i starting after
  // lane i-1's convert) measured 1% slower at 4 lanes, and stream priorities
  // by lane (either order) 7% slower: the gain needs the lanes to co-run.
  int lanes_req = 0;  // 0: auto (3 lanes, 4 from kLanePixels pixels of work)
  static constexpr int kMaxLanes = 4;
  static constexpr int64_t kLanePixels = 24 << 20;  // ~80 VGA frames
  std::vector<Engine*> lane_eng;
  std::vector<cudaStream_t> lane_st;
  std::vector<cudaEvent_t> lane_join;
  cudaEvent_t lane_fork = nullptr;
  int last_lanes = 1;

  bool lanes_off = false;  // automatic lanes ran out of memory once

  int lanes_for(int64_t batch) const {
    if (batch < 2 || (lanes_req == 0 && lanes_off)) return 1;
    int64_t l = lanes_req;
    if (l == 0) {  // auto (tools/probe.py lanes; eager VGA calls: 32 frames ->
                   // 3 lanes +37%, 64 -> 3 lanes +23%, 128 -> 4 lanes +13%,
                   // 256 -> 4 lanes +6%; 3 lanes remain for eager calls < 24 Mpx)
      // graph-replayed calls (<= kGraphMaxBatch frames) split too: the
      // captured graph forks the lanes (VGA x4 0.176 -> 0.155 ms, x8 0.255
      // -> 0.217, x16 0.452 -> 0.344, x32 0.825 -> 0.597, x64 1.339 -> 1.118
      // in 4 lanes)
      const bool big = batch * hw >= kLanePixels;
      if (batch < 4) return 1;
      l = (big || batch <= kGraphMaxBatch) ? kMaxLanes : 3;
    }
    return (int)std::max<int64_t>(1, std::min<int64_t>(l, batch));
  }

  int set_lanes(int n) {
    if (n < 0 || n > 64) {
      set_error("lanes must be in [0, 64] (0 = automatic)");
      return SPX_ERR_VALUE;
    }
    lanes_req = n;
    return SPX_OK;
  }

  int ensure_lanes(int n) {
    SPX_CUDA(cudaSetDevice(device));
    if (!lane_fork) SPX_CUDA(cudaEventCreateWithFlags(&lane_fork, cudaEventDisableTiming));
    const int64_t per = ceil_div(max_batch, (int64_t)n);
    // a lane created for a smaller split cannot take this one's sub-batch;
    // graphs captured over the old children hold their buffer pointers, so
    // every lane graph goes with them (a later call with the same key
    // re-captures over the new children)
    bool replaced = false;
    for (size_t i = 0; i < lane_eng.size(); ++i)
      if (lane_eng[i] && lane_eng[i]->max_batch < per) {
        delete lane_eng[i];
        lane_eng[i] = nullptr;
        replaced = true;
      }
    if (replaced) drop_lane_graphs();
    while ((int)lane_eng.size() < n) {
      lane_eng.push_back(nullptr);
      cudaStream_t q;
      cudaEvent_t e;
      SPX_CUDA(cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking));
      SPX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      lane_st.push_back(q);
      lane_join.push_back(e);
    }
    for (int i = 0; i < n; ++i) {
      if (lane_eng[i]) continue;
      Engine* c = new Engine();
      int rc = c->init(st, per, device);
      if (rc) {
        delete c;
        return rc;
      }
      lane_eng[i] = c;
    }
    return SPX_OK;
  }

  void free_lanes() {
    drop_lane_graphs();
    for (auto c : lane_eng) delete c;
    lane_eng.clear();
    for (auto q : lane_st) cudaStreamDestroy(q);
    for (auto e : lane_join) cudaEventDestroy(e);
    lane_st.clear();
    lane_join.clear();
    if (lane_fork) cudaEventDestroy(lane_fork);
    lane_fork = nullptr;
  }

  int segment_lanes(int n, const uint8_t* rgb, int64_t batch, int32_t* out_labels,
                    double* out_xy, double* out_lab, int64_t* out_counts, int32_t* out_passes,
                    cudaStream_t s) {
    int rc;
    launches = 0;
    n_assoc = n_update = 0;
    stage_mark(ev[EV_START], s);
    SPX_CUDA(cudaEventRecord(lane_fork, s));
    const int64_t per = ceil_div(batch, (int64_t)n);
    int used = 0;
    for (int i = 0; i < n; ++i) {
      const int64_t f0 = i * per, nb = std::min(per, batch - f0);
      if (nb <= 0) break;
      Engine* c = lane_eng[i];
      SPX_CUDA(cudaStreamWaitEvent(lane_st[i], lane_fork, 0));
      // under capture the child records only its start / end events, as
      // event-record nodes (an ordinary record inside a capture would leave
      // the event unusable for a later timing query)
      c->capturing = capturing;
      rc = c->segment_eager(rgb + f0 * hw * 3, nb, out_labels + f0 * hw, out_xy + f0 * K * 2,
                                 out_lab + f0 * K * 3, out_counts + f0 * K,
                                 out_passes ? out_passes + f0 : nullptr, lane_st[i]);
      c->capturing = false;
      if (rc) return rc;
      launches += c->launches;
      SPX_CUDA(cudaEventRecord(lane_join[i], lane_st[i]));
      SPX_CUDA(cudaStreamWaitEvent(s, lane_join[i], 0));
      ++used;
    }
    stage_mark(ev[EV_END], s);
    last_lanes = used;
    return SPX_OK;
  }

  ~Engine() {
    free_lanes();
    cudaSetDevice(device);
    for (void* p : {(void*)lab, (void*)labels, (void*)scratch, (void*)cxy[0], (void*)cxy[1],
                    (void*)clab[0], (void*)clab[1], (void*)slab, (void*)done, (void*)passes,
                    (void*)cc_parent, (void*)cc_size, (void*)cc_nxt, (void*)cc_first,
                    (void*)rec, (void*)acc, (void*)worklist, (void*)sacc, (void*)wwl,
                    (void*)wwl_n})
      if (p) cudaFree(p);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto e : ev_assoc) cudaEventDestroy(e);
    for (auto e : ev_update) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (s_side) cudaStreamDestroy(s_side);
    free_graphs();
    free_staging();
  }

  int init(const spx_settings& s, int64_t mb, int dev) {
    st = s;
    device = dev;
    max_batch = mb;
    SPX_CUDA(cudaSetDevice(dev));
    int major = 0;
    SPX_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major < 10) {
      set_error("device %d has compute capability %d.x; this build targets sm_100a", dev, major);
      return SPX_ERR_CUDA;
    }
    K = st.ns_r * st.ns_c;
    n_bl = ceil_div(3 * st.s, st.tile_len);
    hw = st.width * st.height;
    xy_weight = st.compactness / (double)st.s;  // engine.py:143
    size_t B = (size_t)mb;
    SPX_CUDA(cudaMalloc(&lab, B * plane_of(hw) * 3 * sizeof(float)));
    SPX_CUDA(cudaMalloc(&labels, B * hw * sizeof(int32_t)));
    SPX_CUDA(cudaMalloc(&scratch, B * hw * sizeof(int32_t)));
    for (int i = 0; i < 2; ++i) {
      SPX_CUDA(cudaMalloc(&cxy[i], B * K * 2 * sizeof(double)));
      SPX_CUDA(cudaMalloc(&clab[i], B * K * 3 * sizeof(double)));
      SPX_CUDA(cudaMemset(cxy[i], 0, B * K * 2 * sizeof(double)));
      SPX_CUDA(cudaMemset(clab[i], 0, B * K * 3 * sizeof(double)));
    }
    use_cell = cell_path_ok(st.height, st.width, st.s, st.tile_len) && K < (1ll << 31);
    if (use_cell) {
      SPX_CUDA(cudaMalloc(&rec, B * K * sizeof(CRec)));
      SPX_CUDA(cudaMalloc(&acc, B * K * sizeof(ClusterAcc)));
      SPX_CUDA(cudaMalloc(&worklist, (B * K + 2) * sizeof(int32_t)));
      wl_n = worklist + B * K;
      SPX_CUDA(cudaStreamCreateWithFlags(&s_side, cudaStreamNonBlocking));
      SPX_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      SPX_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
      wide = wide_mode(st.s, st.ns_r, st.ns_c);
      if (wide) {
        const size_t n = B * K * n_bl;
        SPX_CUDA(cudaMalloc(&sacc, n * sizeof(StripAcc)));
        SPX_CUDA(cudaMemset(sacc, 0, n * sizeof(StripAcc)));
        SPX_CUDA(cudaMalloc(&wwl, n * sizeof(long long)));
        SPX_CUDA(cudaMalloc(&wwl_n, sizeof(int32_t)));
        SPX_CUDA(cudaMemset(wwl_n, 0, sizeof(int32_t)));
      }
    } else {
      SPX_CUDA(cudaMalloc(&slab, B * K * n_bl * 6 * sizeof(double)));
    }
    if (st.early_stop >= 0.0) {
      const int rt = shift_tree.build(2 * K, (int)B);
      if (rt) return rt;
    }
    SPX_CUDA(cudaMalloc(&done, B * sizeof(int32_t)));
    SPX_CUDA(cudaMalloc(&passes, B * sizeof(int32_t)));
    if (st.connectivity == 2) {
      SPX_CUDA(cudaMalloc(&cc_parent, B * hw * sizeof(int32_t)));
      SPX_CUDA(cudaMalloc(&cc_size, B * hw * sizeof(int32_t)));
      SPX_CUDA(cudaMalloc(&cc_nxt, B * hw * sizeof(int32_t)));
      SPX_CUDA(cudaMalloc(&cc_first, (B * K + kStrictExtra) * sizeof(int32_t)));
    }
    for (auto& e : ev) SPX_CUDA(cudaEventCreate(&e));
    return SPX_OK;
  }

  cudaEvent_t pass_event(std::vector<cudaEvent_t>& v, size_t i) {
    while (v.size() <= i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      v.push_back(e);
    }
    return v[i];
  }

  // Association pass `pass` (0-based); with_update passes enqueue their
  // flagged clusters into the worklist under count wl_n[pass & 1].
  int associate(int cur, int frames, const int32_t* dn, bool with_update, int pass,
                cudaStream_t s) {
    stage_mark(pass_event(ev_assoc, 2 * n_assoc), s);
    // (wide mode: association only; the update reads the labels itself)
    int rc = use_cell ? launch_cell(lab, cxy[cur], clab[cur], rec, labels, acc, dn, st.height,
                                    st.width, st.s, st.ns_r, st.ns_c, xy_weight, frames,
                                    with_update && !wide, s, 0, -1, 0, worklist,
                                    wl_n + (pass & 1), conc)
                      : launch_assoc(lab, cxy[cur], clab[cur], labels, dn, st.height, st.width,
                                     st.s, st.ns_r, st.ns_c, xy_weight, 0, st.height, frames, K, s);
    stage_mark(pass_event(ev_assoc, 2 * n_assoc + 1), s);
    ++n_assoc;
    ++launches;
    return rc;
  }

  // ---- CUDA graphs ------------------------------------------------------------
  // For small batches (<= kGraphMaxBatch frames) the ~22 launches of a call
  // cost more than the work, so the launch sequence -- which depends only on
  // the batch size and the buffers -- is captured once per (buffers, batch)
  // and replayed with one cudaGraphLaunch (640x480, 1 frame: 292 -> 187 us).
  // The first two calls with a key run eagerly (lazy one-time setup stays out
  // of the graph; the second, warm, call's stage times are kept), the third
  // captures.  Capture uses a private stream (the
  // caller's may be the legacy default stream); replays go on the caller's.
  // Replays record only the start/end events (an event node costs ~4 us);
  // their per-stage breakdown is the one measured on the second eager call.  Large
  // batches run eagerly with every stage event live.
#ifndef SPX_GRAPH_MAX
#define SPX_GRAPH_MAX 64
#endif
  static constexpr int64_t kGraphMaxBatch = SPX_GRAPH_MAX;
  struct GraphEntry {
    const void* key[6];
    int64_t batch;
    int lanes;
    cudaGraphExec_t exec;
    int n_assoc, n_update;
    int64_t launches;
    int eager_calls;
    uint64_t id;
    bool stages_ok;  // `stages` holds this key's warm eager breakdown
    spx_timing stages;
  };
  uint64_t next_graph_id = 1;
  // id of the entry whose second (warm) eager call was the engine's last
  // call: timing() of that call also fills the entry's stage breakdown
  uint64_t stage_pending = 0;
  const GraphEntry* last_graph = nullptr;
  std::vector<GraphEntry> graphs;
  cudaStream_t s_cap = nullptr;
  bool capturing = false;

  // Stage-timing event record.  During capture the external flag turns it
  // into an event-record node of the graph (each replay records the event);
  // otherwise it is an ordinary record.
  // Captured graphs hold no event nodes (SPX_GRAPH_EVENTS=1 restores the
  // start / end nodes): a replay's total comes from ordinary records on the
  // caller's stream around cudaGraphLaunch.
  void stage_mark(cudaEvent_t e, cudaStream_t s) {
    if (capturing) {
      static const bool nodes = getenv("SPX_GRAPH_EVENTS") != nullptr;
      if (!nodes || (e != ev[EV_START] && e != ev[EV_END])) return;
      cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    } else {
      cudaEventRecord(e, s);
    }
  }
  const bool use_graphs = getenv("SPX_NO_GRAPHS") == nullptr;

  // Graph entries whose capture forked into the lane children (lanes > 1).
  void drop_lane_graphs() {
    last_graph = nullptr;
    std::vector<GraphEntry> keep;
    for (auto& g : graphs) {
      if (g.lanes > 1) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
      } else {
        keep.push_back(g);
      }
    }
    graphs.swap(keep);
  }

  void free_graphs() {
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    graphs.clear();
    if (s_cap) cudaStreamDestroy(s_cap);
    s_cap = nullptr;
  }

  int segment(const uint8_t* rgb, int64_t batch, int32_t* out_labels, double* out_xy,
              double* out_lab, int64_t* out_counts, int32_t* out_passes, cudaStream_t s) {
    if (batch < 1 || batch > max_batch) {
      set_error("batch %lld outside [1, %lld]", (long long)batch, (long long)max_batch);
      return SPX_ERR_VALUE;
    }
    SPX_CUDA(cudaSetDevice(device));
    last_graph = nullptr;
    const uint64_t prev_pending = stage_pending;
    stage_pending = 0;
    int nl = lanes_for(batch);
    if (nl > 1) {
      const int rl = ensure_lanes(nl);
      // Automatic lanes whose child buffers do not fit next to the caller's
      // tensors: give the memory back and run unsplit from now on (same
      // results, same kernels).  An explicit lane count reports the error.
      if (rl != SPX_OK) {
        if (rl != SPX_ERR_NOMEM || lanes_req != 0) return rl;
        free_lanes();
        cudaGetLastError();
        lanes_off = true;
        nl = 1;
      }
    }
    // one call, eager: unsplit or in lanes (the lanes' buffers exist by now)
    auto run = [&](cudaStream_t q) {
      if (nl > 1)
        return segment_lanes(nl, rgb, batch, out_labels, out_xy, out_lab, out_counts, out_passes,
                             q);
      last_lanes = 1;
      return segment_eager(rgb, batch, out_labels, out_xy, out_lab, out_counts, out_passes, q);
    };
    if (!use_graphs || batch > kGraphMaxBatch) return run(s);
    const void* key[6] = {rgb, out_labels, out_xy, out_lab, out_counts, out_passes};
    GraphEntry* g = nullptr;
    for (auto& e : graphs)
      if (e.batch == batch && e.lanes == nl && std::memcmp(e.key, key, sizeof key) == 0) g = &e;
    if (!g) {  // first call with this key: eager, remember the key
      if (graphs.size() >= 8) {
        if (graphs.front().exec) cudaGraphExecDestroy(graphs.front().exec);
        graphs.erase(graphs.begin());
      }
      GraphEntry e{};
      std::memcpy(e.key, key, sizeof key);
      e.batch = batch;
      e.lanes = nl;
      e.eager_calls = 1;
      e.id = next_graph_id++;
      graphs.push_back(e);
      return run(s);
    }
    if (!g->exec && g->eager_calls < 2) {  // second call: eager and warm
      ++g->eager_calls;
      const int rc = run(s);
      if (rc == SPX_OK) stage_pending = g->id;
      return rc;
    }
    if (!g->exec) {  // third call: capture
      // The stage breakdown replays report is the warm eager call's: taken
      // by timing() if the caller asked for it, else here when that call
      // was this engine's last one (its events are still the newest).  An
      // interleaved key in between leaves the breakdown unknown (zeros;
      // replays still measure their total).
      if (!g->stages_ok && prev_pending == g->id) {
        int rt = timing(&g->stages);
        if (rt) return rt;
        g->stages_ok = true;
      }
      if (!s_cap) SPX_CUDA(cudaStreamCreateWithFlags(&s_cap, cudaStreamNonBlocking));
      SPX_CUDA(cudaStreamBeginCapture(s_cap, cudaStreamCaptureModeRelaxed));
      capturing = true;
      int rc = run(s_cap);
      capturing = false;
      cudaGraph_t graph = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(s_cap, &graph);
      if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      if (ce != cudaSuccess) {
        set_error("graph capture failed: %s", cudaGetErrorString(ce));
        return SPX_ERR_CUDA;
      }
      const cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) {
        g->exec = nullptr;
        set_error("graph instantiate failed: %s", cudaGetErrorString(ie));
        return SPX_ERR_CUDA;
      }
      g->n_assoc = n_assoc;
      g->n_update = n_update;
      g->launches = launches;
    }
    static const bool nodes = getenv("SPX_GRAPH_EVENTS") != nullptr;
    if (!nodes) SPX_CUDA(cudaEventRecord(ev[EV_START], s));
    SPX_CUDA(cudaGraphLaunch(g->exec, s));
    if (!nodes) SPX_CUDA(cudaEventRecord(ev[EV_END], s));
    n_assoc = g->n_assoc;
    n_update = g->n_update;
    launches = g->launches;
    last_graph = g;
    last_lanes = g->lanes;
    return SPX_OK;
  }

  int segment_eager(const uint8_t* rgb, int64_t batch, int32_t* out_labels, double* out_xy,
                    double* out_lab, int64_t* out_counts, int32_t* out_passes, cudaStream_t s) {
    const int B = (int)batch;
    const bool early = st.early_stop >= 0.0;
    int rc;
    n_assoc = n_update = 0;
    launches = 0;
    const int32_t* dn = early ? done : nullptr;
    stage_mark(ev[EV_START], s);
    // (wide mode: the flag marks pixels outside the strip-level range)
    if ((rc = launch_convert(rgb, lab, 0, (int64_t)B * hw, st.color_space, s, use_cell ? hw : 0,
                             st.s, wide ? strip_tau(st.s, st.tile_len) : -1.f)))
      return rc;
    ++launches;
    stage_mark(ev[EV_CONVERT], s);
    // The last init launch also writes the fp32 records (cell path), clears
    // the accumulators and zeroes the two worklist counts.
    CRec* i_rec = use_cell ? rec : nullptr;
    ClusterAcc* i_acc = use_cell ? acc : nullptr;
    int32_t* i_zero = use_cell ? wl_n : nullptr;
    const int i_nz = use_cell ? 2 : 0;
    const bool pert = st.perturb;
    if ((rc = launch_init(lab, st.height, st.width, st.s, st.ns_c, cxy[0], clab[0], 0, K, K, B, 0,
                          1, s, use_cell, -1, 0, pert ? nullptr : i_rec, pert ? nullptr : i_acc,
                          pert ? nullptr : i_zero, pert ? 0 : i_nz)))
      return rc;
    ++launches;
    stage_mark(ev[EV_INIT], s);
    if (pert) {
      if ((rc = launch_init(lab, st.height, st.width, st.s, st.ns_c, cxy[0], clab[0], 0, K, K, B,
                            1, 0, s, use_cell, -1, 0, i_rec, i_acc, i_zero, i_nz)))
        return rc;
      ++launches;
    }
    stage_mark(ev[EV_PERTURB], s);
    if (early) {
      SPX_CUDA(cudaMemsetAsync(passes, 0, B * sizeof(int32_t), s));
      SPX_CUDA(cudaMemsetAsync(done, 0, B * sizeof(int32_t), s));
    }
    int cur = 0, nxt = 1;
    if ((rc = associate(cur, B, dn, true, 0, s))) return rc;
    for (int it = 0; it < st.no_iters; ++it) {
      stage_mark(pass_event(ev_update, 2 * n_update), s);
      if (use_cell && wide) {
        if ((rc = launch_wide_update(lab, labels, sacc, wwl, wwl_n, cxy[cur], clab[cur],
                                     cxy[nxt], clab[nxt], out_counts, rec, dn, st.height,
                                     st.width, st.s, st.ns_r, st.ns_c, st.tile_len, B, s)))
          return rc;
        launches += 3;
      } else if (use_cell && merged_update) {
        // reduce + exact fallback of pass `it`'s worklist as one launch
        // (k_update; the reduce also zeroes the next pass's count)
        if ((rc = launch_reduce_cells(acc, lab, labels, cxy[cur], clab[cur], cxy[nxt], clab[nxt],
                                      out_counts, rec, dn, worklist, wl_n + (it & 1), st.height,
                                      st.width, st.s, st.ns_r, st.ns_c, st.tile_len, B, s, 0, -1,
                                      0, kReduceExactMerged, wl_n + ((it + 1) & 1))))
          return rc;
        launches += 1;
      } else if (use_cell) {
        // fork: the exact fallback (pass `it`'s worklist) on the side stream,
        // the reduce (which also zeroes the next pass's count) here; join
        SPX_CUDA(cudaEventRecord(ev_fork, s));
        SPX_CUDA(cudaStreamWaitEvent(s_side, ev_fork, 0));
        if ((rc = launch_reduce_cells(acc, lab, labels, cxy[cur], clab[cur], cxy[nxt], clab[nxt],
                                      out_counts, rec, dn, worklist, wl_n + (it & 1), st.height,
                                      st.width, st.s, st.ns_r, st.ns_c, st.tile_len, B, s_side,
                                      0, -1, 0, kExactOnly)))
          return rc;
        SPX_CUDA(cudaEventRecord(ev_join, s_side));
        if ((rc = launch_reduce_cells(acc, lab, labels, cxy[cur], clab[cur], cxy[nxt], clab[nxt],
                                      out_counts, rec, dn, worklist, wl_n + (it & 1), st.height,
                                      st.width, st.s, st.ns_r, st.ns_c, st.tile_len, B, s, 0, -1,
                                      0, kReduceOnly, wl_n + ((it + 1) & 1))))
          return rc;
        SPX_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
        launches += 2;
      } else {
        if ((rc = launch_accum_range(lab, labels, st.height, st.width, slab, n_bl, st.s, st.ns_c,
                                     st.tile_len, 0, K, K, B, dn, s)))
          return rc;
        if ((rc = launch_reduce(slab, n_bl, cxy[cur], clab[cur], cxy[nxt], clab[nxt], out_counts,
                                0, K, K, B, dn, s)))
          return rc;
        launches += 2;
      }
      stage_mark(pass_event(ev_update, 2 * n_update + 1), s);
      ++n_update;
      if (early) {
        // shift + per-frame pass count (engine.py:196); flags early stop
        if ((rc = shift_tree.launch(cxy[nxt], cxy[cur], 2 * K, B, nullptr, done, passes,
                                    st.early_stop, s)))
          return rc;
        ++launches;
      }
      std::swap(cur, nxt);
      const bool more = it + 1 < st.no_iters;
      if ((rc = associate(cur, B, dn, more, it + 1, s))) return rc;
      if (early) {
        if ((rc = launch_commit_done(done, B, s))) return rc;
        ++launches;
      }
    }
    stage_mark(ev[EV_CONN0], s);
    // Final centres: frame f ends in buffer passes[f] & 1 (ping-pong,
    // engine.py:197; without early stop every frame ran no_iters passes).
    // The same launch writes the per-frame pass counts.  It only needs the
    // finished update passes, so on the cell path it runs on the side stream
    // beside the connectivity pass (joined before the end event).
    cudaStream_t sg = use_cell ? s_side : s;
    if (use_cell) {
      SPX_CUDA(cudaEventRecord(ev_fork, s));
      SPX_CUDA(cudaStreamWaitEvent(s_side, ev_fork, 0));
    }
    k_gather_centres<<<(unsigned)ceil_div(K * B, 256), 256, 0, sg>>>(
        cxy[0], clab[0], cxy[1], clab[1], early ? passes : nullptr, early ? -1 : (int)st.no_iters,
        K, B, out_xy, out_lab, out_passes);
    SPX_LAUNCH_CHECK("k_gather_centres");
    ++launches;
    if (use_cell) SPX_CUDA(cudaEventRecord(ev_join, s_side));
    if (st.connectivity == 1) {
      if ((rc = launch_weak2(labels, out_labels, st.height, st.width, B, s, 0, -1))) return rc;
      ++launches;
    } else if (st.connectivity == 2) {
      if ((rc = launch_strict(labels, out_labels, st.height, st.width, B, K, st.min_size,
                              cc_parent, cc_size, cc_nxt, cc_first, s)))
        return rc;
      int rounds = 1;  // k_cc_local, border, resolve, first, next, jump x (rounds + 1), write
      while ((1ll << rounds) < hw) ++rounds;
      launches += 6 + rounds + 1;
    } else {
      SPX_CUDA(cudaMemcpyAsync(out_labels, labels, (size_t)B * hw * sizeof(int32_t),
                               cudaMemcpyDeviceToDevice, s));
    }
    if (use_cell) SPX_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
    stage_mark(ev[EV_END], s);
    return SPX_OK;
  }

  int timing(spx_timing* t) {
    SPX_CUDA(cudaSetDevice(device));
    SPX_CUDA(cudaEventSynchronize(ev[EV_END]));
    std::memset(t, 0, sizeof *t);
    auto el = [](cudaEvent_t a, cudaEvent_t b) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      return ms;
    };
    if (last_graph) {  // graph replay: measured total, eager-call breakdown
      *t = last_graph->stages;
      t->total = el(ev[EV_START], ev[EV_END]);
      return SPX_OK;
    }
    if (last_lanes > 1) {  // lanes: lane 0's stages (run concurrently), measured total
      int rc = lane_eng[0]->timing(t);
      if (rc) return rc;
      t->total = el(ev[EV_START], ev[EV_END]);
      keep_pending_stages(*t);
      return SPX_OK;
    }
    t->convert = el(ev[EV_START], ev[EV_CONVERT]);
    t->init = el(ev[EV_CONVERT], ev[EV_INIT]);
    t->perturb = el(ev[EV_INIT], ev[EV_PERTURB]);
    t->connectivity = el(ev[EV_CONN0], ev[EV_END]);
    t->total = el(ev[EV_START], ev[EV_END]);
    t->n_associate = std::min(n_assoc, 1024);
    t->n_update = std::min(n_update, 1024);
    for (int i = 0; i < t->n_associate; ++i) t->associate[i] = el(ev_assoc[2 * i], ev_assoc[2 * i + 1]);
    for (int i = 0; i < t->n_update; ++i) t->update[i] = el(ev_update[2 * i], ev_update[2 * i + 1]);
    keep_pending_stages(*t);
    return SPX_OK;
  }

  void keep_pending_stages(const spx_timing& t) {
    if (!stage_pending) return;
    for (auto& g : graphs)
      if (g.id == stage_pending && !g.stages_ok) {
        g.stages = t;
        g.stages_ok = true;
      }
    stage_pending = 0;
  }

  // ---- host-buffer entry point: chunked, triple-buffered, three streams -------
  // H2D of chunk c+1 and D2H of chunk c-1 overlap the compute of chunk c
  // (copy engines run both directions concurrently with the SMs).  Host
  // buffers must be pinned for the copies to be asynchronous; pageable
  // buffers still give correct results, serialised.
  int64_t chunk = 0, chunk_req = 64;
  // Three staging slots: the compute of chunk c reuses chunk c-3's slot, so
  // it never waits for the previous chunk's download (which, sharing PCIe
  // with the next upload, is the longest of the three stages).
  static constexpr int kSlots = 3;
  uint8_t* h_rgb[kSlots] = {};
  uint8_t* h_out[kSlots] = {};  // one block per slot, carved by out_layout(nb)
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_h2d[kSlots] = {}, ev_comp[kSlots] = {}, ev_d2h[kSlots] = {};

  // Byte offsets of the five outputs of `nb` frames in one block (256-byte
  // aligned): labels, cxy, clab, counts, passes, total.  A caller whose host
  // outputs follow the same layout (spx_engine_output_layout) gets one D2H
  // copy per chunk instead of five.
  void out_layout(int64_t nb, int64_t* o) const {
    auto al = [](int64_t v) { return (v + 255) & ~(int64_t)255; };
    o[0] = 0;
    o[1] = al(nb * hw * 4);
    o[2] = o[1] + al(nb * K * 16);
    o[3] = o[2] + al(nb * K * 24);
    o[4] = o[3] + al(nb * K * 8);
    o[5] = o[4] + nb * 4;
  }

  int ensure_staging() {
    if (s_comp) return SPX_OK;
    chunk = std::max<int64_t>(1, std::min<int64_t>(max_batch, chunk_req));
    int64_t lay[6];
    out_layout(chunk, lay);
    for (int i = 0; i < kSlots; ++i) {
      SPX_CUDA(cudaMalloc(&h_rgb[i], chunk * hw * 3));
      SPX_CUDA(cudaMalloc(&h_out[i], lay[5]));
      SPX_CUDA(cudaEventCreateWithFlags(&ev_h2d[i], cudaEventDisableTiming));
      SPX_CUDA(cudaEventCreateWithFlags(&ev_comp[i], cudaEventDisableTiming));
      SPX_CUDA(cudaEventCreateWithFlags(&ev_d2h[i], cudaEventDisableTiming));
    }
    SPX_CUDA(cudaStreamCreateWithFlags(&s_h2d, cudaStreamNonBlocking));
    SPX_CUDA(cudaStreamCreateWithFlags(&s_comp, cudaStreamNonBlocking));
    SPX_CUDA(cudaStreamCreateWithFlags(&s_d2h, cudaStreamNonBlocking));
    return SPX_OK;
  }

  void free_staging() {
    for (int i = 0; i < kSlots; ++i) {
      for (void* q : {(void*)h_rgb[i], (void*)h_out[i]})
        if (q) cudaFree(q);
      for (cudaEvent_t e : {ev_h2d[i], ev_comp[i], ev_d2h[i]})
        if (e) cudaEventDestroy(e);
      h_rgb[i] = nullptr, h_out[i] = nullptr;
      ev_h2d[i] = ev_comp[i] = ev_d2h[i] = nullptr;
    }
    for (auto& r : subs) {
      if (r.a) cudaEventDestroy(r.a);
      if (r.b) cudaEventDestroy(r.b);
      r = SubRec();
    }
    for (cudaStream_t q : {s_h2d, s_comp, s_d2h})
      if (q) cudaStreamDestroy(q);
    s_h2d = s_comp = s_d2h = nullptr;
  }

  // Frames per pipeline chunk.  Small chunks expose less fill/drain in a single
  // call; chunk = batch is best for a stream of batches (bench: 256).
  int set_host_chunk(int64_t n) {
    if (n < 1) {
      set_error("host chunk must be >= 1");
      return SPX_ERR_VALUE;
    }
    int rc = wait_host();
    if (rc) return rc;
    free_staging();
    chunk_req = n;
    seq = 0;
    return SPX_OK;
  }

  // Host-buffer pipeline: chunks of `chunk` frames alternate between two
  // device staging slots; H2D, compute and D2H run on three streams ordered
  // by events.  The slot sequence continues across calls, so back-to-back
  // submit_host calls (a stream of batches) keep all three engines busy and
  // only the very first H2D and the last D2H are exposed.
  int64_t seq = 0;
  std::vector<cudaEvent_t> tl;  // SPX_DEBUG_TIMELINE=1 per-chunk timeline
  // Device time of each submission (compute stream: first chunk's start to
  // last chunk's end), kept for the last kSubRing submissions so a consumer
  // of batch i can read its time without waiting for batch i+1.
  static constexpr int kSubRing = 8;
  struct SubRec {
    int64_t ticket = 0;
    cudaEvent_t a = nullptr, b = nullptr;
  } subs[kSubRing];
  int64_t n_subs = 0;

  // `sync`: the caller waits for this call right away (segment_host).  A
  // one-chunk synchronous call then runs H2D, compute and D2H on the compute
  // stream alone (no cross-stream event hops: one 640x480 frame's call is
  // latency-bound), still ordered after earlier submissions of the slot.
  int submit_host(const uint8_t* rgb, int64_t batch, int32_t* out_labels, double* out_xy,
                  double* out_lab, int64_t* out_counts, int32_t* out_passes, bool sync = false) {
    SPX_CUDA(cudaSetDevice(device));
    int rc = ensure_staging();
    if (rc) return rc;
    if (batch < 1) {
      set_error("batch must be >= 1");
      return SPX_ERR_VALUE;
    }
    const int64_t nchunks = ceil_div(batch, chunk);
    const bool one_stream = sync && nchunks == 1;
    cudaStream_t q_h2d = one_stream ? s_comp : s_h2d, q_d2h = one_stream ? s_comp : s_d2h;
    // host outputs laid out as one block (spx_engine_output_layout): one D2H
    int64_t hl[6];
    out_layout(batch, hl);
    const char* hb = reinterpret_cast<const char*>(out_labels);
    const bool host_block = nchunks == 1 && out_labels &&
                            reinterpret_cast<const char*>(out_xy) == hb + hl[1] &&
                            reinterpret_cast<const char*>(out_lab) == hb + hl[2] &&
                            reinterpret_cast<const char*>(out_counts) == hb + hl[3] &&
                            reinterpret_cast<const char*>(out_passes) == hb + hl[4];
    SubRec& sr = subs[n_subs % kSubRing];
    if (!sr.a) {
      SPX_CUDA(cudaEventCreate(&sr.a));
      SPX_CUDA(cudaEventCreate(&sr.b));
    }
    static const bool dbg = getenv("SPX_DEBUG_TIMELINE") != nullptr;
    auto mark = [&](cudaStream_t q) {
      if (!dbg) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, q);
      tl.push_back(e);
    };
    for (int64_t c = 0; c < nchunks; ++c, ++seq) {
      const int sl = (int)(seq % kSlots);
      const int64_t f0 = c * chunk, nb = std::min(chunk, batch - f0);
      int64_t lay[6];
      out_layout(nb, lay);
      uint8_t* ob = h_out[sl];
      int32_t* d_lab = reinterpret_cast<int32_t*>(ob + lay[0]);
      double* d_xy = reinterpret_cast<double*>(ob + lay[1]);
      double* d_cl = reinterpret_cast<double*>(ob + lay[2]);
      int64_t* d_cnt = reinterpret_cast<int64_t*>(ob + lay[3]);
      int32_t* d_pass = reinterpret_cast<int32_t*>(ob + lay[4]);
      if (seq >= kSlots) SPX_CUDA(cudaStreamWaitEvent(q_h2d, ev_comp[sl], 0));
      if (seq >= kSlots && one_stream) SPX_CUDA(cudaStreamWaitEvent(s_comp, ev_d2h[sl], 0));
      mark(q_h2d);
      SPX_CUDA(cudaMemcpyAsync(h_rgb[sl], rgb + f0 * hw * 3, nb * hw * 3, cudaMemcpyHostToDevice,
                               q_h2d));
      mark(q_h2d);
      if (!one_stream) {
        SPX_CUDA(cudaEventRecord(ev_h2d[sl], s_h2d));
        SPX_CUDA(cudaStreamWaitEvent(s_comp, ev_h2d[sl], 0));
        if (seq >= kSlots) SPX_CUDA(cudaStreamWaitEvent(s_comp, ev_d2h[sl], 0));
      }
      // (a synchronous one-stream call needs no events: the host waits for
      // it before any later submission can reuse the slot)
      if (c == 0 && !one_stream) SPX_CUDA(cudaEventRecord(sr.a, s_comp));
      mark(s_comp);
      if ((rc = segment(h_rgb[sl], nb, d_lab, d_xy, d_cl, d_cnt, d_pass, s_comp))) return rc;
      mark(s_comp);
      if (c == nchunks - 1 && !one_stream) SPX_CUDA(cudaEventRecord(sr.b, s_comp));
      if (!one_stream) SPX_CUDA(cudaEventRecord(ev_comp[sl], s_comp));
      if (!one_stream) SPX_CUDA(cudaStreamWaitEvent(s_d2h, ev_comp[sl], 0));
      mark(q_d2h);
      if (host_block) {
        SPX_CUDA(cudaMemcpyAsync(out_labels, ob, lay[5], cudaMemcpyDeviceToHost, q_d2h));
      } else {
        if (out_labels)
          SPX_CUDA(cudaMemcpyAsync(out_labels + f0 * hw, d_lab, nb * hw * 4,
                                   cudaMemcpyDeviceToHost, q_d2h));
        if (out_xy)
          SPX_CUDA(cudaMemcpyAsync(out_xy + f0 * K * 2, d_xy, nb * K * 16,
                                   cudaMemcpyDeviceToHost, q_d2h));
        if (out_lab)
          SPX_CUDA(cudaMemcpyAsync(out_lab + f0 * K * 3, d_cl, nb * K * 24,
                                   cudaMemcpyDeviceToHost, q_d2h));
        if (out_counts)
          SPX_CUDA(cudaMemcpyAsync(out_counts + f0 * K, d_cnt, nb * K * 8,
                                   cudaMemcpyDeviceToHost, q_d2h));
        if (out_passes)
          SPX_CUDA(cudaMemcpyAsync(out_passes + f0, d_pass, nb * 4, cudaMemcpyDeviceToHost,
                                   q_d2h));
      }
      mark(q_d2h);
      if (!one_stream) SPX_CUDA(cudaEventRecord(ev_d2h[sl], q_d2h));
    }
    if (!one_stream) {
      sr.ticket = seq;
      ++n_subs;
    }
    last_sync = one_stream;
    return SPX_OK;
  }
  bool last_sync = false;

  // Compute-stream time (ms) of the submission that returned `ticket`; waits
  // for that submission's compute only.
  int ticket_time(int64_t ticket, float* ms) {
    SPX_CUDA(cudaSetDevice(device));
    for (auto& r : subs)
      if (r.a && r.ticket == ticket && ticket > 0) {
        SPX_CUDA(cudaEventSynchronize(r.b));
        SPX_CUDA(cudaEventElapsedTime(ms, r.a, r.b));
        return SPX_OK;
      }
    set_error("no timing kept for ticket %lld (the last %d submissions are kept)",
              (long long)ticket, kSubRing);
    return SPX_ERR_VALUE;
  }

  // Wait for the submissions up to `ticket` (a value of `seq` after a submit).
  // A slot's event may since have been re-recorded by a later chunk; waiting
  // on it is still correct (the D2H stream is in order), only later.
  int wait_ticket(int64_t ticket) {
    SPX_CUDA(cudaSetDevice(device));
    if (ticket <= 0 || !s_d2h) return SPX_OK;
    if (ticket > seq) {
      set_error("ticket %lld was never issued", (long long)ticket);
      return SPX_ERR_VALUE;
    }
    SPX_CUDA(cudaEventSynchronize(ev_d2h[(ticket - 1) % kSlots]));
    return SPX_OK;
  }

  int wait_host() {
    SPX_CUDA(cudaSetDevice(device));
    if (!s_d2h) return SPX_OK;
    SPX_CUDA(cudaStreamSynchronize(s_d2h));
    SPX_CUDA(cudaStreamSynchronize(s_comp));  // one-stream calls end there
    if (!tl.empty()) {
      for (size_t i = 0; i + 5 < tl.size(); i += 6) {
        float a0, a1, b0, b1, c0, c1;
        cudaEventElapsedTime(&a0, tl[0], tl[i]);
        cudaEventElapsedTime(&a1, tl[0], tl[i + 1]);
        cudaEventElapsedTime(&b0, tl[0], tl[i + 2]);
        cudaEventElapsedTime(&b1, tl[0], tl[i + 3]);
        cudaEventElapsedTime(&c0, tl[0], tl[i + 4]);
        cudaEventElapsedTime(&c1, tl[0], tl[i + 5]);
        fprintf(stderr, "chunk %zu: h2d %.2f-%.2f comp %.2f-%.2f d2h %.2f-%.2f ms\n", i / 6, a0, a1,
                b0, b1, c0, c1);
      }
      for (auto e : tl) cudaEventDestroy(e);
      tl.clear();
    }
    return SPX_OK;
  }

  int segment_host(const uint8_t* rgb, int64_t batch, int32_t* out_labels, double* out_xy,
                   double* out_lab, int64_t* out_counts, int32_t* out_passes) {
    int rc = submit_host(rgb, batch, out_labels, out_xy, out_lab, out_counts, out_passes, true);
    int rw = wait_host();
    return rc ? rc : rw;
  }
};

}  // namespace spx

struct spx_engine {
  spx::Engine e;
};

extern "C" {

int32_t spx_engine_create(const spx_settings* st, int64_t max_batch, int32_t device,
                          spx_engine** out) {
  using namespace spx;
  *out = nullptr;
  if (!st || st->width < 1 || st->height < 1 || st->s < 1 || st->ns_r < 1 || st->ns_c < 1 ||
      st->no_iters < 1 || st->tile_len < 1 || !(st->compactness > 0) || st->min_size < 1) {
    set_error("invalid engine settings");
    return SPX_ERR_INVALID_SETTINGS;
  }
  if ((st->height - 1) / st->s >= st->ns_r || (st->width - 1) / st->s >= st->ns_c) {
    set_error("grid %lldx%lld at s=%lld does not cover %lldx%lld", (long long)st->ns_c,
              (long long)st->ns_r, (long long)st->s, (long long)st->width, (long long)st->height);
    return SPX_ERR_INVALID_SETTINGS;
  }
  if (st->color_space < 0 || st->color_space > 2 || st->connectivity < 0 || st->connectivity > 2) {
    set_error("invalid colour space / connectivity code");
    return SPX_ERR_INVALID_SETTINGS;
  }
  if (max_batch < 1 || max_batch > 65535) {
    set_error("max_batch must be in [1, 65535]");
    return SPX_ERR_VALUE;
  }
  spx_engine* eng = new spx_engine();
  int rc = eng->e.init(*st, max_batch, device);
  if (rc) {
    delete eng;
    return rc;
  }
  *out = eng;
  return SPX_OK;
}

int32_t spx_engine_destroy(spx_engine* eng) {
  delete eng;
  return SPX_OK;
}

int32_t spx_engine_segment(spx_engine* eng, const uint8_t* rgb_dev, int64_t batch,
                           int32_t* labels_dev, double* cxy_dev, double* clab_dev,
                           int64_t* counts_dev, int32_t* passes_dev, void* stream) {
  return eng->e.segment(rgb_dev, batch, labels_dev, cxy_dev, clab_dev, counts_dev, passes_dev,
                        spx::as_stream(stream));
}

int32_t spx_engine_segment_host(spx_engine* eng, const uint8_t* rgb_host, int64_t batch,
                                int32_t* labels_host, double* cxy_host, double* clab_host,
                                int64_t* counts_host, int32_t* passes_host) {
  return eng->e.segment_host(rgb_host, batch, labels_host, cxy_host, clab_host, counts_host,
                             passes_host);
}

int32_t spx_engine_submit_host(spx_engine* eng, const uint8_t* rgb_host, int64_t batch,
                               int32_t* labels_host, double* cxy_host, double* clab_host,
                               int64_t* counts_host, int32_t* passes_host) {
  return eng->e.submit_host(rgb_host, batch, labels_host, cxy_host, clab_host, counts_host,
                            passes_host);
}

int32_t spx_engine_wait(spx_engine* eng) { return eng->e.wait_host(); }

int64_t spx_engine_ticket(spx_engine* eng) { return eng->e.seq; }

int32_t spx_engine_wait_ticket(spx_engine* eng, int64_t ticket) {
  return eng->e.wait_ticket(ticket);
}

int32_t spx_engine_output_layout(spx_engine* eng, int64_t batch, int64_t* out6) {
  if (batch < 1) {
    spx::set_error("batch must be >= 1");
    return SPX_ERR_VALUE;
  }
  eng->e.out_layout(batch, out6);
  return SPX_OK;
}

int32_t spx_engine_ticket_time(spx_engine* eng, int64_t ticket, float* ms) {
  return eng->e.ticket_time(ticket, ms);
}

int32_t spx_engine_set_host_chunk(spx_engine* eng, int64_t frames) {
  return eng->e.set_host_chunk(frames);
}

int32_t spx_engine_timing(spx_engine* eng, spx_timing* out) { return eng->e.timing(out); }

int32_t spx_engine_set_lanes(spx_engine* eng, int32_t lanes) { return eng->e.set_lanes(lanes); }

int32_t spx_engine_last_lanes(spx_engine* eng) { return eng->e.last_lanes; }

int64_t spx_engine_last_launches(spx_engine* eng) { return eng->e.launches; }

int32_t spx_engine_fused_path(spx_engine* eng) { return eng->e.use_cell ? 1 : 0; }

}  // extern "C"
