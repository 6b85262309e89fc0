// Host runtime + C ABI: communicators, flag memory, CUDA-IPC peer mappings,
// symmetric registration, staging, CTA/channel assignment and launches.
//
// Two process models share one device executor (exec.cu):
//   single-process (blink_init_all): all ranks' buffers are visible to one
//     host thread.  Calls are batched until every rank of the comm set has
//     called (implicit NCCL-style group); then one cooperative launch per
//     device runs the channels of all ranks on that device.  Ranks may share
//     a device ("virtual ranks": their HBM stands in for the peers' HBM).
//   multi-process (blink_init + export/connect): one rank per process; peers'
//     flags, staging and registered buffers are CUDA-IPC mappings over
//     NVLink/NVSwitch; each call launches this rank's channels only, with an
//     entry handshake and an exit wait.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <mutex>
#include <thread>
#include <chrono>
#include <numeric>
#include <tuple>
#include <string>
#include <unistd.h>
#include <sys/syscall.h>
#include <cerrno>
#ifndef SYS_pidfd_open
#define SYS_pidfd_open 434
#endif
#ifndef SYS_pidfd_getfd
#define SYS_pidfd_getfd 438
#endif
#include <vector>

#include "blink_internal.h"

using namespace blink;

namespace {

thread_local std::string g_last_error;

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

struct SizedKey {
  int coll, root, dtype;
  size_t count;
  uint64_t launch_mask;
  size_t chunk = 0;  // MIAD override (0 = static table)
  bool operator<(const SizedKey& o) const {
    if (chunk != o.chunk) return chunk < o.chunk;
    if (coll != o.coll) return coll < o.coll;
    if (root != o.root) return root < o.root;
    if (dtype != o.dtype) return dtype < o.dtype;
    if (count != o.count) return count < o.count;
    return launch_mask < o.launch_mask;
  }
};

struct Sized {
  const Plan* plan = nullptr;
  std::vector<TreeRange> ranges;
  std::vector<DevTask> tasks;
  DevTask* d_tasks = nullptr;
  DevTree* d_trees = nullptr;
  std::vector<DevTree> htrees;  // host copy (kernel parameters)
  bool merged_all = false;      // every CTA runs tasks[0] with its own index
  int64_t mchunk = 0, mbytes = 0;  // merged: byte-range chunks over the whole buffer
  int ctas = 0;
  int chunks = 0;
  int nctr = 0;  // dynamic chunk counters used by the launch
  int chan0 = 0, nchan = 0;  // work stealing: channel descriptors after the CTAs' tasks
  bool lsu = false;          // small chunks: the register (LSU) path, not the TMA pipeline
};

struct Reg {
  char* buf = nullptr;
  size_t bytes = 0;
  char* peer[kMaxRanks] = {};
};

struct Clique;

struct Pending {
  bool posted = false;
  const void* send = nullptr;
  void* recv = nullptr;
  cudaStream_t stream = nullptr;
};

}  // namespace

struct blink_comm {
  int nranks = 0, rank = 0, device = 0;
  blink_config_t cfg{};
  Graph graph;
  bool multiprocess = false;
  bool connected = false;
  Clique* clique = nullptr;
  uint64_t calls = 0;  // multi-process: collectives launched (epochs live on the device)
  uint64_t* flags = nullptr;  // kFlagBytes of flag words, then ll_bytes of LL areas
  uint64_t* peer_flags[kMaxRanks] = {};
  size_t ll_bytes = 0;
  std::map<std::pair<size_t, int>, std::vector<int64_t>> ll_lo;  // LL slices per (count, esize)
  int* err_host = nullptr;  // multi-process error word
  int* err_dev = nullptr;
  uint64_t* ctrl = nullptr;  // multi-process: device launch epoch + done counter
  int sms = 148;
  std::map<std::pair<int, int>, std::unique_ptr<Plan>> plans;  // (coll, root|variant)
  std::map<SizedKey, Sized> sized;                             // multi-process launches
  std::vector<Reg> regs;
  std::map<std::string, char*> opened;  // peer IPC handle bytes -> mapped base
  char* staging = nullptr;
  size_t staging_bytes = 0;
  char* peer_staging[kMaxRanks] = {};
  // NEXT-1: multicast-bound buffer (uc/mc mappings) when NVLS is on
  NvlsMem nvls;
  bool nvls_on = false;
  std::string nvls_note = "off (cfg.nvls = 0)";
  std::vector<int> exported_fds;      // VMM registration: fds peers duplicate (closed at destroy)
  std::vector<VmmMapping> vmm_maps;   // VMM registration: peers' chunks mapped here
  Probe probe;                // topology probe result (graph == NULL at init)
  bool probe_at_connect = false;  // multi-process: graph == NULL, probed from the peers' bus ids
  char* scratch = nullptr;    // single-process Gather on link graphs: forwarding buffer of a
  size_t scratch_bytes = 0;   // rank that passed recvbuf == NULL but relays other blocks
  std::string last_error;
  blink_stats_t stats{};
  // multi-process MIAD (NEXT-2): rank 0 decides each autotuned call's chunk
  // size and publishes it in its flag words; the other ranks read it there
  struct MpMiad {
    blink_miad_t st{};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool pending = false;  // rank 0: ev0/ev1 bracket a launch not yet folded into st
    bool done = false;     // converged (phase 2) and published: no more slots
    size_t chunk = 0;      // chunk of the last autotuned call (identical on every rank)
    int calls = 0;
  };
  std::map<std::tuple<int, int, int, size_t>, MpMiad> mp_miad;  // (coll, root, dtype, count)
  uint64_t miad_seq = 0;                // autotuned calls so far (same sequence on every rank)
  cudaStream_t miad_stream = nullptr;   // non-blocking stream for reading rank 0's slots
};

namespace {

struct Clique {
  std::mutex mu;
  int nranks = 0;
  bool nvls = false;         // NEXT-1 active (one rank per device, multicast object bound)
  std::vector<blink_comm*> comms;
  std::vector<int> devices;  // distinct devices
  // launch groups: the ranks one launch runs.  One group per device (ranks
  // sharing a device are batched), or one per rank with cfg.launch_per_rank.
  // Error words, control words and traces are keyed by the group key.
  struct Group {
    int key, device;
    uint64_t mask;
  };
  std::vector<Group> groups;
  bool per_rank = false;
  std::vector<cudaStream_t> rstream;  // per_rank: rank v's library-owned launch stream
  std::vector<cudaEvent_t> rfork, rjoin;
  int alive = 0;
  uint64_t calls = 0;  // batches launched (epochs live on the device)
  // the batch being assembled
  int nposted = 0;
  int coll = -1, root = -1, dtype = -1, op = -1;
  size_t count = 0;
  std::vector<Pending> pending;
  // per launch group state
  std::map<int, int*> err_host, err_dev;
  std::map<int, uint64_t*> ctrl;  // per group: launch epoch + done counter
  std::map<int, uint64_t*> trace; // per group: BLINK_TRACE stamps of the last launch
  std::map<int, int> trace_ctas;
  struct MiadRun {
    blink_miad_t st;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool pending = false;
    int calls = 0;  // the first call (plan + table build) is not timed
  };
  std::map<std::tuple<int, int, int, size_t>, MiadRun> miad;  // (coll, root, dtype, count)
  std::map<SizedKey, Sized> sized;
  int64_t launches = 0;
};

blink_result_t fail(blink_comm_t comm, blink_result_t r, const std::string& msg) {
  g_last_error = msg;
  if (comm) comm->last_error = msg;
  if (getenv("BLINK_DEBUG")) fprintf(stderr, "[blink] error %d: %s\n", int(r), msg.c_str());
  return r;
}

#define CUDA_TRY(comm, call)                                                          \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(comm, BLINK_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

blink_config_t resolve_cfg(const blink_config_t* c) {
  blink_config_t d;
  blink_config_default(&d);
  blink_config_t tmp;
  if (!c) {
    tmp = d;
    c = &tmp;
  }
  blink_config_t r = *c;
  // environment overrides (tuning): BLINK_THREADS, BLINK_CTAS, BLINK_CHUNK_BYTES
  if (const char* e = getenv("BLINK_THREADS")) r.threads = atoi(e);
  if (const char* e = getenv("BLINK_CTAS")) r.ctas = atoi(e);
  if (const char* e = getenv("BLINK_CHUNK_BYTES")) r.chunk_bytes = size_t(atoll(e));
  if (const char* e = getenv("BLINK_MIAD")) r.autotune = atoi(e);
  if (const char* e = getenv("BLINK_PER_RANK")) r.launch_per_rank = atoi(e);
  if (const char* e = getenv("BLINK_LL_MAX")) r.ll_max_bytes = size_t(atoll(e));
  if (const char* e = getenv("BLINK_SHALLOW_MAX")) r.shallow_max_bytes = size_t(atoll(e));
  if (const char* e = getenv("BLINK_NVLS")) r.nvls = atoi(e);
  if (r.nvls_bytes == 0) r.nvls_bytes = d.nvls_bytes;
  r.nvls_bytes = (r.nvls_bytes + 15) / 16 * 16;
  if (r.ll_max_bytes > (size_t(16) << 20)) r.ll_max_bytes = size_t(16) << 20;
  r.ll_max_bytes = r.ll_max_bytes / kGrain * kGrain;
  if (!(r.mwu_eps > 0 && r.mwu_eps < 1)) r.mwu_eps = d.mwu_eps;
  if (!(r.ilp_gap > 0 && r.ilp_gap < 1)) r.ilp_gap = d.ilp_gap;
  if (r.threads <= 0) r.threads = d.threads;
  if (r.threads > 256) r.threads = 256;  // __launch_bounds__(256, 1)
  if (r.threads < 128) r.threads = 128;  // producer + store + >= 2 consumer warps
  r.threads = (r.threads + 31) / 32 * 32;
  if (!(r.timeout_s > 0)) r.timeout_s = d.timeout_s;
  if (r.staging_bytes == 0) r.staging_bytes = d.staging_bytes;
  r.staging_bytes = (r.staging_bytes + 4095) / 4096 * 4096;
  return r;
}

// Plan cache: key (coll, root) with root = -1 for AllReduce, root + 1000
// for the one-hop Broadcast star variant on switches, root + 2000 for the
// single minimum-depth tree of small calls on link graphs (R#27).
blink_result_t get_plan(blink_comm_t comm, int coll, int root, size_t bytes, const Plan** out) {
  int key_root = (coll == kBroadcast || coll == kGather) ? root : -1;
  if (is_block_coll(coll) && comm->graph.multi_server)
    return fail(comm, BLINK_ERR_UNSUPPORTED, "multi-server graphs support AllReduce only");
  const bool link_blocks = is_block_coll(coll) && !comm->graph.switch_model;  // NEXT-3 on link graphs
  bool star = coll == kBroadcast && comm->graph.switch_model && comm->nranks > 2 &&
              bytes <= comm->cfg.onehop_bcast_max_bytes;
  if (star) key_root += 1000;
  const bool shallow = !is_block_coll(coll) && use_shallow_plan(comm->graph, coll, bytes, comm->cfg);
  if (shallow) key_root += 2000;
  auto k = std::make_pair(coll, key_root);
  auto it = comm->plans.find(k);
  if (it != comm->plans.end()) {
    *out = it->second.get();
    return BLINK_SUCCESS;
  }
  auto p = std::make_unique<Plan>();
  std::string err;
  blink_result_t r;
  if (star) {
    p->coll = kBroadcast;
    p->root = root;
    p->nranks = comm->nranks;
    p->switch_model = true;
    Tree t;
    t.root = root;
    t.parent.assign(comm->nranks, root);
    t.parent[root] = -1;
    t.depth = 1;
    p->trees.push_back(t);
    p->rate_num = 1;
    r = BLINK_SUCCESS;
  } else if (shallow) {
    r = make_shallow_plan(comm->graph, coll, root, p.get(), &err);
  } else if (link_blocks) {
    r = make_block_plan(comm->graph, coll, root, p.get(), &err);
  } else {
    r = make_plan(comm->graph, is_block_coll(coll) ? kAllReduce : coll, root, comm->cfg, p.get(),
                  &err);
    if (is_block_coll(coll)) {  // one-hop stars; tree j owns block j
      p->coll = coll;
      p->blocks = true;
      if (coll == kGather)  // star j keeps the single leaf `root`
        for (Tree& t : p->trees)
          for (int v = 0; v < int(t.parent.size()); ++v)
            if (t.parent[v] >= 0 && v != root) t.parent[v] = -2;
    }
  }
  if (r != BLINK_SUCCESS) return fail(comm, r, err);
  if (getenv("BLINK_DEBUG")) {
    std::vector<TreeRange> none;
    fprintf(stderr, "[blink] plan %s\n", plan_to_json(*p, 0, 4, none, 0).c_str());
  }
  *out = p.get();
  comm->plans[k] = std::move(p);
  return BLINK_SUCCESS;
}

bool steal_on();
int64_t lsu_chunk_max();

struct Channel {
  int rank, tree, role, parent;
  uint32_t children, leafmask;
  double work;
  int ctas = 1;
};

// Channels of the ranks in `mask` and their CTA shares of `budget` (a6):
// CTAs in proportion to bytes x operands.  Returns false (with *err) when the
// channels do not fit the budget.  *nexit = ranks in `mask` without a channel.
bool alloc_channels(const Plan& plan, const std::vector<std::vector<uint32_t>>& ch,
                    const std::vector<TreeRange>& r0, int esize, uint64_t mask, int budget,
                    std::vector<Channel>* out, int* nexit_out, std::string* err) {
  const int n = plan.nranks;
  const int k = int(plan.trees.size());
  std::vector<Channel>& chans = *out;
  chans.clear();
  std::vector<int> rank_has(n, 0);
  for (int v = 0; v < n; ++v) {
    if (!((mask >> v) & 1)) continue;
    for (int i = 0; i < k; ++i) {
      uint32_t c = ch[i][v];
      const bool own_block = plan.blocks && is_push_coll(plan.coll) && plan.trees[i].root == v;
      if (!c && !own_block) continue;
      int nc = __builtin_popcount(c);
      uint32_t leaf = 0;
      for (int u = 0; u < n; ++u)
        if (((c >> u) & 1u) && ch[i][u] == 0) leaf |= 1u << u;
      double bytes = double(r0[i].hi - r0[i].lo) * esize + 1.0;
      int par = plan.trees[i].parent[v];
      if (plan.coll == kAllReduce) {
        double wr = bytes * ((nc + 1) + (par < 0 ? nc + 1 : 1));
        chans.push_back({v, i, kRoleReduce, par, c, leaf, wr});
        if (par >= 0) chans.push_back({v, i, kRoleBcast, par, c, leaf, bytes * (1 + nc)});
      } else if (plan.coll == kReduceScatter) {
        chans.push_back({v, i, kRoleReduce, par, c, leaf, bytes * (nc + 2)});
      } else {
        chans.push_back({v, i, kRoleBcast, par, c, leaf, bytes * (1 + nc + (par < 0 ? 1 : 0))});
      }
      rank_has[v] = 1;
    }
  }
  int nexit = 0;
  for (int v = 0; v < n; ++v)
    if (((mask >> v) & 1) && !rank_has[v]) ++nexit;
  *nexit_out = nexit;
  const int avail = budget - nexit;
  if (int(chans.size()) > avail) {
    *err = "plan needs " + std::to_string(chans.size() + nexit) + " channels but only " +
           std::to_string(budget) + " CTAs can be co-resident";
    return false;
  }
  // Proportional split: CTAs in proportion to work, largest remainders get
  // the CTAs the floors left over (every SM works); ties by channel order, so
  // every launch group computes the same split.
  double tot = 0;
  for (auto& c : chans) tot += c.work;
  int used = 0;
  std::vector<std::pair<double, int>> rem;  // (fractional share, channel)
  for (size_t j = 0; j < chans.size(); ++j) {
    Channel& c = chans[j];
    const double share = avail * c.work / tot;
    c.ctas = std::max(1, int(std::floor(share)));
    rem.push_back({share - std::floor(share), int(j)});
    used += c.ctas;
  }
  std::stable_sort(rem.begin(), rem.end(),
                   [](const std::pair<double, int>& a, const std::pair<double, int>& b) { return a.first > b.first; });
  for (size_t j = 0; used < avail && j < rem.size(); ++j, ++used) ++chans[rem[j].second].ctas;
  while (used > avail) {  // trim the largest
    auto it = std::max_element(chans.begin(), chans.end(),
                               [](const Channel& a, const Channel& b) { return a.ctas < b.ctas; });
    --it->ctas;
    --used;
  }
  // Makespan split: every channel starts with one CTA and each further CTA
  // goes to the channel with the most work per CTA (ties: channel order).
  // It minimises max(work / ctas), the slowest channel's time, over integer
  // splits.  With dozens of channels on one device (multi-level trees of
  // virtual ranks) the proportional split rounds shares of 1-2 CTAs to 1 or
  // 2, up to 2x between the channels of one tree (DGX-1V AllReduce 256 MiB:
  // 1-CTA channels ended at 1.85 ms, others at 0.61 ms).  It replaces the
  // proportional split only when that rounding leaves the slowest channel
  // >= 10% slower; with large shares the two differ by one CTA here and there
  // and the proportional split measured as fast or faster.
  // BLINK_ALLOC=prop|greedy forces one.
  static const int mode = [] {
    const char* e = getenv("BLINK_ALLOC");
    if (!e) return 0;
    return std::string(e) == "prop" ? 1 : (std::string(e) == "greedy" ? 2 : 0);
  }();
  if (mode == 1 || chans.empty()) return true;
  std::vector<int> g(chans.size(), 1);
  for (int u = int(chans.size()); u < avail; ++u) {
    size_t best = 0;
    for (size_t j = 1; j < chans.size(); ++j)
      if (chans[j].work * g[best] > chans[best].work * g[j]) best = j;
    ++g[best];
  }
  double mp = 0, mg = 0;
  for (size_t j = 0; j < chans.size(); ++j) {
    mp = std::max(mp, chans[j].work / chans[j].ctas);
    mg = std::max(mg, chans[j].work / g[j]);
  }
  if (mode == 2 || mg < 0.9 * mp)
    for (size_t j = 0; j < chans.size(); ++j) chans[j].ctas = g[j];
  if (getenv("BLINK_DEBUG_TASKS"))
    fprintf(stderr, "[blink] alloc: %zu channels, %d CTAs, makespan prop %.4g greedy %.4g -> %s\n",
            chans.size(), avail, mp, mg, (mode == 2 || mg < 0.9 * mp) ? "greedy" : "prop");
  return true;
}

// CTA / channel assignment for the ranks in `launch_mask` (a6) and the device
// tables of one launch.  `group_masks` lists every launch group of the call
// (one per process, device or rank); the chunking must be the same in all of
// them, because a chunk's flags name the same bytes on every rank, so the
// chunk-size hints come from all groups' channel shares, not this group's.
blink_result_t build_sized(blink_comm_t comm, const Plan& plan, size_t count, int esize,
                           uint64_t launch_mask, const std::vector<uint64_t>& group_masks,
                           int budget, Sized* s, size_t chunk_override = 0) {
  blink_config_t cfg = comm->cfg;
  if (chunk_override) cfg.chunk_bytes = chunk_override;
  const int n = plan.nranks;
  const int k = int(plan.trees.size());
  std::vector<std::vector<uint32_t>> ch(k, std::vector<uint32_t>(n, 0));
  for (int i = 0; i < k; ++i)
    for (int v = 0; v < n; ++v)
      if (plan.trees[i].parent[v] >= 0) ch[i][plan.trees[i].parent[v]] |= 1u << v;
  // provisional byte shares (equal CTAs hint) to weigh channels
  std::vector<TreeRange> r0;
  std::string err;
  blink_result_t rr = size_plan(plan, count, esize, cfg, 1, &r0, &err);
  if (rr != BLINK_SUCCESS) return fail(comm, rr, err);
  std::vector<Channel> chans;
  int nexit = 0;
  if (!alloc_channels(plan, ch, r0, esize, launch_mask, budget, &chans, &nexit, &err))
    return fail(comm, BLINK_ERR_UNSUPPORTED, err);
  // chunk-size hint per tree: the busiest channel of the tree in any group
  std::vector<int> hint(k, 1);
  for (uint64_t gm : group_masks) {
    std::vector<Channel> gch;
    int gx = 0;
    if (gm == launch_mask) {
      gch = chans;
    } else if (!alloc_channels(plan, ch, r0, esize, gm, budget, &gch, &gx, &err)) {
      return fail(comm, BLINK_ERR_UNSUPPORTED, err);
    }
    for (auto& c : gch) hint[c.tree] = std::max(hint[c.tree], c.ctas);
  }
  // ---- merged one-hop AllReduce (single launch): every tree's root channel
  // reads every rank's send and writes every rank's recv, so one channel over
  // the concatenated chunks of all trees, fed by one dynamic counter, uses
  // every co-resident CTA and balances them to the last chunk.
  {
    const uint64_t all = (n >= 64) ? ~uint64_t(0) : ((uint64_t(1) << n) - 1);
    const uint32_t allm = uint32_t(all);
    bool mergeable = launch_mask == all && plan.coll == kAllReduce && !chans.empty() &&
                     !(getenv("BLINK_MERGE") && getenv("BLINK_MERGE")[0] == '0');
    for (auto& c : chans)
      mergeable = mergeable && c.role == kRoleReduce && c.parent < 0 && c.leafmask == c.children &&
                  (c.children | (1u << c.rank)) == allm;
    if (mergeable && int(chans.size()) == k) {
      const int B = budget;
      std::vector<TreeRange> ri;
      if (size_plan(plan, count, esize, cfg, std::max(1, B / k), &ri, &err) != BLINK_SUCCESS)
        return fail(comm, BLINK_ERR_INTERNAL, err);
      s->ranges = ri;
      // Every tree here is a star over all ranks with the same operand order
      // (ascending ranks), so a byte's result does not depend on which tree
      // holds it: the merged channel cuts the whole buffer into chunks of the
      // trees' (largest) chunk size -- the chunk-to-bytes map is arithmetic.
      int64_t cb = 0;
      for (auto& r : ri) cb = std::max<int64_t>(cb, r.chunk * int64_t(esize));
      cb = std::max<int64_t>(cb, kGrain);
      const int64_t S = int64_t(count) * esize;
      const int64_t per = std::max<int64_t>(1, (S + int64_t(B) * cb - 1) / (int64_t(B) * cb));
      if (cfg.chunk_bytes == 0 && per <= 8) {
        // medium calls (<= 8 chunks per CTA): the static table's chunk,
        // shrunk so that about the same number of chunks goes to every CTA
        // (1 MiB runs on all SMs instead of S / 16 KiB of them; no one-chunk
        // tail), in 1 KiB steps (tile-friendly sizes), not below 4 KiB.
        // A/B, m = 8 per call: 256 KiB 7.6 -> 6.0 us, 1 MiB 7.8 -> 6.8 us
        // up to 4 chunks per CTA (8 with <= 4 ranks): one larger chunk per
        // CTA instead -- fewer chunk set-ups and drains, and the per-call
        // ramp overlaps better (A/B per call: m = 8 3/4/6 MiB 10.7/11.6/17.4
        // -> 9.4/10.7/16.7 us; m = 4 8 MiB 13.3 -> 11.7 us; m = 2 6/16 MiB
        // 9.3/15.0 -> 7.4/11.7 us; beyond these limits, or above 192 KiB
        // per chunk, it loses)
        static const int one_env = [] {
          const char* e = getenv("BLINK_ONE_CHUNK");
          return e ? atoi(e) : -1;
        }();
        const int64_t one_max = one_env >= 0 ? one_env : (n <= 4 ? 8 : 4);
        const int64_t one_bytes = (S + int64_t(B) - 1) / int64_t(B);  // <= 192 KiB (m = 2 48 MiB: 7% slower)
        const int64_t per2 = (per >= 2 && per <= one_max && one_bytes <= (192 << 10)) ? 1 : per;
        int64_t c2 = (S + int64_t(B) * per2 - 1) / (int64_t(B) * per2);
        c2 = (c2 + 1023) / 1024 * 1024;
        cb = per2 < per ? c2 : std::max<int64_t>(std::min<int64_t>(c2, cb), std::min<int64_t>(cb, 4 << 10));
      }
      const int total = int((S + cb - 1) / cb);
      s->mchunk = cb;
      s->mbytes = S;
      const int ctas = std::max(1, std::min(B, total));
      s->tasks.assign(ctas, DevTask{});
      for (int j = 0; j < ctas; ++j) {
        DevTask& t = s->tasks[j];
        t.rank = 0;
        t.tree = 0;
        t.role = kRoleReduce;
        t.parent = -1;
        t.children = allm & ~1u;
        t.leafmask = allm & ~1u;
        t.cta_idx = j;
        t.cta_cnt = ctas;
        t.exit_cnt = 1;
        t.next = -1;
        t.c0 = j;
        t.c1 = total;
        t.cstride = ctas;
        t.ctr = 0;
        t.merged = 1;
      }
      s->nctr = 1;
      s->ctas = ctas;
      s->chunks = total;
      s->plan = &plan;
      s->merged_all = true;
      // the merged one-hop AllReduce is latency-bound below a few MiB too: the
      // register path (every thread loads all m operands, combines, stores)
      // skips the pipeline's ramp (BLINK_LSU_MERGED_MAX bytes per rank)
      static const int64_t merged_max = [] {
        const char* e = getenv("BLINK_LSU_MERGED_MAX");
        return e ? int64_t(atoll(e)) : (int64_t(4) << 20);
      }();
      s->lsu = lsu_chunk_max() > 0 && S <= merged_max;
      return BLINK_SUCCESS;
    }
  }
  // ---- packed assignment (opt-in, BLINK_PACK=1; measured no faster than the
  // per-channel split on the 1-GPU bench): one launch holding every rank whose channels are
  // independent (no chunk-level waits: one-hop roots) and equally loaded.
  // Every CTA gets the same number of chunks as a contiguous range of the
  // global chunk list, possibly spanning two trees (chained segments).
  {
    bool packable = launch_mask == ((n >= 64) ? ~uint64_t(0) : ((uint64_t(1) << n) - 1)) &&
                    !chans.empty() && cfg.chunk_bytes == 0 && getenv("BLINK_PACK") != nullptr;
    for (auto& c : chans) {
      const bool indep =
          c.parent < 0 && ((c.role == kRoleReduce && c.leafmask == c.children) ||
                           (c.role == kRoleBcast && (plan.coll == kBroadcast || plan.coll == kAllGather)));
      packable = packable && indep && std::fabs(c.work - chans[0].work) <= 1e-3 * chans[0].work + 64;
    }
    const int B = budget;
    const int nch = int(chans.size());
    if (packable) {
      const int g = std::gcd(nch, B);
      const int per = B * (nch / g) / nch;  // chunks per channel; total = B * (nch / g)
      const int64_t tbytes = (r0[chans[0].tree].hi - r0[chans[0].tree].lo) * esize;
      int64_t chunk = ((tbytes + per - 1) / per + kGrain - 1) / kGrain * kGrain;
      if (per <= kMaxChunks && chunk >= (4 << 10)) {
        blink_config_t c2 = cfg;
        c2.chunk_bytes = size_t(chunk);
        std::vector<TreeRange> ri;
        if (size_plan(plan, count, esize, c2, 1, &ri, &err) != BLINK_SUCCESS)
          return fail(comm, BLINK_ERR_INTERNAL, err);
        s->ranges = ri;
        // global chunk list: channel-major
        std::vector<std::pair<int, int>> items;  // (channel, chunk)
        for (int ci = 0; ci < nch; ++ci)
          for (int c = 0; c < s->ranges[chans[ci].tree].nchunks; ++c) items.push_back({ci, c});
        const int64_t T = int64_t(items.size());
        s->tasks.assign(B, DevTask{});
        std::vector<DevTask> extra;
        std::vector<int> entry_done(n, 0);
        auto mk = [&](int ci, int c0, int c1) {
          const Channel& ch = chans[ci];
          DevTask t{};
          t.rank = int16_t(ch.rank);
          t.tree = int16_t(ch.tree);
          t.role = int16_t(ch.role);
          t.parent = int16_t(ch.parent);
          t.children = ch.children;
          t.leafmask = ch.leafmask;
          t.c0 = c0;
          t.c1 = c1;
          t.cstride = 1;
          t.ctr = -1;
          t.cta_cnt = 1;
          t.exit_cnt = 1;
          t.next = -1;
          if (!entry_done[ch.rank]) {
            t.do_entry = 1;
            entry_done[ch.rank] = 1;
          }
          return t;
        };
        for (int k = 0; k < B; ++k) {
          const int64_t a0 = k * T / B, a1 = (k + 1) * T / B;
          std::vector<DevTask> segs;
          int64_t i = a0;
          while (i < a1) {
            const int ci = items[i].first;
            int64_t j = i;
            while (j < a1 && items[j].first == ci) ++j;
            segs.push_back(mk(ci, items[i].second, items[j - 1].second + 1));
            i = j;
          }
          if (segs.empty()) {  // more CTAs than chunks: an idle CTA
            DevTask t{};
            t.role = kRoleExit;
            t.parent = -1;
            t.cta_cnt = 1;
            t.exit_cnt = 1;
            t.next = -1;
            t.ctr = -1;
            segs.push_back(t);
          }
          s->tasks[k] = segs[0];
          int* link = &s->tasks[k].next;
          for (size_t q = 1; q < segs.size(); ++q) {
            *link = B + int(extra.size());
            extra.push_back(segs[q]);
            link = &extra.back().next;
          }
        }
        // ranks without a channel still publish their entry (chained on CTA 0)
        for (int v = 0; v < n; ++v) {
          if (entry_done[v]) continue;
          DevTask t{};
          t.rank = int16_t(v);
          t.role = kRoleExit;
          t.parent = -1;
          t.cta_cnt = 1;
          t.exit_cnt = 1;
          t.do_entry = 1;
          t.ctr = -1;
          t.next = s->tasks[0].next;
          s->tasks[0].next = B + int(extra.size());
          extra.push_back(t);
        }
        s->tasks.insert(s->tasks.end(), extra.begin(), extra.end());
        s->ctas = B;
        s->chunks = int(T);
        s->plan = &plan;
        return BLINK_SUCCESS;
      }
    }
  }
  // chunking with the CTA count of the busiest channel of each tree (hint)
  s->ranges.clear();
  for (int i = 0; i < k; ++i) {
    std::vector<TreeRange> ri;
    rr = size_plan(plan, count, esize, cfg, hint[i], &ri, &err);
    if (rr != BLINK_SUCCESS) return fail(comm, rr, err);
    s->ranges.push_back(ri[i]);
  }
  for (auto& c : chans) c.ctas = std::max(1, std::min(c.ctas, s->ranges[c.tree].nchunks));
  // tasks: grouped by rank so exit work is split across a rank's CTAs
  s->tasks.clear();
  s->chunks = 0;
  for (auto& r : s->ranges) s->chunks += r.nchunks;
  const bool dynamic = !(getenv("BLINK_DYNAMIC") && getenv("BLINK_DYNAMIC")[0] == '0') &&
                       int(chans.size()) <= kMaxCounters;
  s->nctr = dynamic ? int(chans.size()) : 0;
  for (int v = 0; v < n; ++v) {
    if (!((launch_mask >> v) & 1)) continue;
    size_t first = s->tasks.size();
    for (size_t ci = 0; ci < chans.size(); ++ci) {
      const Channel& c = chans[ci];
      if (c.rank != v) continue;
      for (int j = 0; j < c.ctas; ++j) {
        DevTask t{};
        t.rank = int16_t(v);
        t.tree = int16_t(c.tree);
        t.role = int16_t(c.role);
        t.parent = int16_t(c.parent);
        t.children = c.children;
        t.leafmask = c.leafmask;
        t.cta_idx = j;
        t.cta_cnt = c.ctas;
        t.next = -1;
        t.c0 = j;
        t.c1 = s->ranges[c.tree].nchunks;
        t.cstride = c.ctas;
        t.ctr = dynamic ? int(ci) : -1;
        s->tasks.push_back(t);
      }
    }
    if (s->tasks.size() == first) {
      DevTask t{};
      t.rank = int16_t(v);
      t.role = kRoleExit;
      t.parent = -1;
      t.cta_cnt = 1;
      t.next = -1;
      t.ctr = -1;
      s->tasks.push_back(t);
    }
    int cnt = int(s->tasks.size() - first);
    for (int j = 0; j < cnt; ++j) {
      s->tasks[first + j].exit_idx = j;
      s->tasks[first + j].exit_cnt = cnt;
      s->tasks[first + j].do_entry = (j == 0);
    }
  }
  s->ctas = int(s->tasks.size());
  s->plan = &plan;
  // Small chunks run the register path: one hop of a chunk through the TMA
  // pipeline (flag -> producer warp -> bulk load -> mbarrier -> store warp ->
  // bulk store -> drain -> flag) takes 3.5 us at 4 KiB, the all-threads LSU
  // copy 1.6 us (scripts/hop_probe.py), and per-CTA throughput only matters
  // once chunks are large (A/B per call, 1 MiB: DGX-1V Broadcast 23.6 -> 16.9
  // us, 3-GPU chains 11.1 -> 8.0, switch two-level Broadcast 13.1 -> 10.4,
  // DGX-1V AllReduce 37.9 -> 33.6; 4 MiB even; TMA wins from 16 MiB).
  // One-hop plans (stars: ReduceScatter / AllGather blocks, per-rank
  // launches) keep 16 KiB chunks at every size, so there it also needs few
  // chunks per CTA (<= 4, the latency regime): ReduceScatter 16 / 64 MiB ran
  // 31 / 96 us on the TMA pipeline and 51 / 173 us on the register path.
  {
    int64_t maxc = 0;
    int depth = 0, per = 0;
    for (auto& r : s->ranges) maxc = std::max<int64_t>(maxc, r.chunk * int64_t(esize));
    for (auto& t : plan.trees) depth = std::max(depth, t.depth);
    for (auto& c : chans)
      if ((launch_mask >> c.rank) & 1)
        per = std::max(per, (s->ranges[c.tree].nchunks + c.ctas - 1) / c.ctas);
    // Only calls of <= 1.5 MiB per rank (BLINK_LSU_SMALL_CALL): since the
    // pipeline's proxy fences were narrowed (3.6 -> 3.2 us per hop) it is as
    // fast or faster from 2 MiB, while the register path still wins 5-20% at
    // 0.25-1.5 MiB, chunks up to 96 KiB (ab_lsu_small_r02.txt)
    static const int64_t small_call = [] {
      const char* e = getenv("BLINK_LSU_SMALL_CALL");
      return e ? int64_t(atoll(e)) : (int64_t(3) << 19);
    }();
    const int64_t cap = lsu_chunk_max();
    s->lsu = cap > 0 && int64_t(count) * esize <= small_call && maxc <= cap && (depth >= 2 || per <= 4);
  }
  // work stealing (a6): one descriptor per dynamic channel after the CTAs'
  // tasks.  A CTA whose own chunks are all taken joins the channel with the
  // most chunks left; it takes chunks from that channel's counter only
  // (cta_idx = -1), so a channel's chunks still go out in increasing order.
  // Only when some channel has more than 3 rounds of chunks for its own CTAs
  // (a CTA joins a channel with > 2 rounds left): otherwise nobody can join,
  // and the exit-time scan would only delay the last CTA (about 1 us).
  bool stealable = false;
  for (auto& c : chans)
    stealable = stealable || (((launch_mask >> c.rank) & 1) && s->ranges[c.tree].nchunks > 3 * c.ctas);
  if (dynamic && steal_on() && stealable && !s->lsu) {
    s->chan0 = int(s->tasks.size());
    for (size_t ci = 0; ci < chans.size(); ++ci) {
      if (!((launch_mask >> chans[ci].rank) & 1)) continue;
      for (int j = 0; j < s->chan0; ++j) {
        if (s->tasks[j].ctr != int(ci)) continue;
        DevTask t = s->tasks[j];
        t.cta_idx = -1;
        t.do_entry = 0;
        t.next = -1;
        s->tasks.push_back(t);
        break;
      }
    }
    s->nchan = int(s->tasks.size()) - s->chan0;
  }
  if (getenv("BLINK_DEBUG_TASKS")) {  // CTA -> channel map (scripts/trace_tree.py)
    for (size_t j = 0; j < size_t(s->ctas); ++j) {
      const DevTask& t = s->tasks[j];
      fprintf(stderr, "[blink] cta %zu rank %d tree %d role %d parent %d children %x chunks %d\n", j,
              int(t.rank), int(t.tree), int(t.role), int(t.parent), t.children, t.c1);
    }
  }
  return BLINK_SUCCESS;
}

// Switches this thread's stream-capture mode to relaxed for its lifetime:
// allocations and uploads made on behalf of a call being captured into a CUDA
// graph are not part of the graph and must not invalidate the capture.
struct RelaxedCapture {
  cudaStreamCaptureMode prev = cudaStreamCaptureModeRelaxed;
  RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&prev); }
  ~RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&prev); }
};

blink_result_t finalize_tables(blink_comm_t comm, int device, int esize, Sized* s) {
  DeviceGuard g(device);
  std::vector<DevTree> trees(s->ranges.size());
  for (size_t i = 0; i < s->ranges.size(); ++i) {
    trees[i].lo = s->ranges[i].lo * esize;
    trees[i].hi = s->ranges[i].hi * esize;
    trees[i].chunk = s->ranges[i].chunk * esize;
    trees[i].nchunks = s->ranges[i].nchunks;
    trees[i].root = s->plan->trees[i].root;
    uint32_t mem = 0;
    for (size_t v = 0; v < s->plan->trees[i].parent.size(); ++v)
      if (s->plan->trees[i].parent[v] != -2) mem |= 1u << v;
    trees[i].members = mem;
  }
  for (auto& t : s->tasks)
    if (t.tree >= 0 && size_t(t.tree) < trees.size()) t.tr = trees[t.tree];
  s->htrees = trees;
  // a call first seen while its stream is being captured into a CUDA graph
  // builds its tables here too: allocate and upload outside the capture
  // (relaxed mode, a private non-blocking stream) so the capture stays valid
  RelaxedCapture rc;
  CUDA_TRY(comm, cudaMalloc(&s->d_tasks, sizeof(DevTask) * s->tasks.size()));
  CUDA_TRY(comm, cudaMalloc(&s->d_trees, sizeof(DevTree) * std::max<size_t>(1, trees.size())));
  cudaStream_t up = nullptr;
  CUDA_TRY(comm, cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
  cudaError_t e = cudaMemcpyAsync(s->d_tasks, s->tasks.data(), sizeof(DevTask) * s->tasks.size(),
                                  cudaMemcpyHostToDevice, up);
  if (e == cudaSuccess && !trees.empty())
    e = cudaMemcpyAsync(s->d_trees, trees.data(), sizeof(DevTree) * trees.size(), cudaMemcpyHostToDevice, up);
  if (e == cudaSuccess) e = cudaStreamSynchronize(up);
  cudaStreamDestroy(up);
  CUDA_TRY(comm, e);
  return BLINK_SUCCESS;
}

// Data path: BLINK_TMA=0 register/LSU loads and stores, 1 TMA loads + LSU
// stores, 2 TMA loads + TMA bulk stores (default).
// Launch attributes.  Default: programmatic dependent launch (PDL) -- a
// call's kernel is launched while the previous kernel in the stream drains,
// and waits (griddepcontrol.wait) before touching memory: 1.2-2.6 us less per
// back-to-back eager call (scripts/pdl_probe.cu).  PDL gains nothing on a
// cooperative launch, so co-residency then rests on the grid sizing (grid <=
// occupancy x SMs, co_resident_budget) as it does for per-rank launches and
// NCCL's kernels.  BLINK_PDL=0 launches cooperatively instead (the driver
// checks co-residency); BLINK_COOP=0 with BLINK_PDL=0 sets neither.
bool use_pdl() {
  static bool v = [] {
    const char* e = getenv("BLINK_PDL");
    return !(e && e[0] == '0');
  }();
  return v;
}
bool use_coop() {
  static bool v = [] {
    const char* e = getenv("BLINK_COOP");
    return !use_pdl() && !(e && e[0] == '0');
  }();
  return v;
}

int use_tma() {
  static int v = [] {
    const char* e = getenv("BLINK_TMA");
    if (!e || !e[0]) return 2;
    return e[0] == '0' ? 0 : (e[0] == '1' ? 1 : 2);
  }();
  return v;
}

// Shared-memory ring size and tile (tuning knobs; defaults from bench sweeps).
int smem_bytes() {
  static int v = [] {
    const char* e = getenv("BLINK_SMEM_KB");
    int kb = e ? atoi(e) : 200;
    if (kb < 16) kb = 16;
    if (kb > 224) kb = 224;
    return kb * 1024;
  }();
  return v;
}
int store_depth() {
  static int v = [] {
    const char* e = getenv("BLINK_STORE_DEPTH");
    return e ? atoi(e) : -1;
  }();
  return v;
}
// Largest chunk that runs the register path in a non-merged launch
// (BLINK_LSU_CHUNK_MAX bytes; 0 = always the TMA pipeline).
int64_t lsu_chunk_max() {
  static int64_t v = [] {
    const char* e = getenv("BLINK_LSU_CHUNK_MAX");
    return e ? int64_t(atoll(e)) : int64_t(96 << 10);
  }();
  return v;
}
// Work stealing across a launch's channels (default on; BLINK_STEAL=0 off).
bool steal_on() {
  static bool v = [] {
    const char* e = getenv("BLINK_STEAL");
    return !(e && e[0] == '0');
  }();
  return v;
}
int copy_stages() {
  static int v = [] {
    const char* e = getenv("BLINK_COPY_STAGES");
    return e ? atoi(e) : 0;
  }();
  return v;
}
int split_ring() {
  static int v = [] {
    const char* e = getenv("BLINK_SPLIT_RING");
    return e ? atoi(e) : 1;
  }();
  return v;
}
int l2_hint() {
  static int v = [] {
    const char* e = getenv("BLINK_L2HINT");
    return e ? atoi(e) : 0;
  }();
  return v;
}
// deferred chunk signals (exec.cu run_ws); BLINK_DEFER_SIGNAL=0 drains per chunk
int defer_signal() {
  static int v = [] {
    const char* e = getenv("BLINK_DEFER_SIGNAL");
    return e ? atoi(e) : 1;
  }();
  return v;
}
int tile_bytes() {
  static int v = [] {
    const char* e = getenv("BLINK_TILE");
    int t = e ? atoi(e) : 0;
    return t > 0 ? (t + 15) / 16 * 16 : 0;
  }();
  return v;
}

int co_resident_budget(blink_comm_t comm, int device, int dtype, int op, int coll) {
  DeviceGuard g(device);
  int per_sm = exec_max_ctas_per_sm(comm->cfg.threads, true, dtype, op, coll, smem_bytes());
  int per_sm2 = exec_max_ctas_per_sm(comm->cfg.threads, false, dtype, op, coll, 0);
  per_sm = std::min(per_sm, per_sm2);
  if (per_sm <= 0) per_sm = 1;
  int cap = per_sm * comm->sms;
  if (comm->cfg.ctas > 0) cap = std::min(cap, comm->cfg.ctas);
  return cap;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

blink_result_t validate_call(blink_comm_t comm, size_t count, blink_dtype_t dtype, int op,
                             int root, int coll) {
  if (!comm) return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "comm is NULL");
  if (esize_of(dtype) == 0)
    return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "unsupported dtype " + std::to_string(dtype));
  if ((coll == kAllReduce || coll == kReduceScatter) && (op < BLINK_SUM || op > BLINK_AVG))
    return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "unsupported op " + std::to_string(op));
  if ((coll == kBroadcast || coll == kGather) && (root < 0 || root >= comm->nranks))
    return fail(comm, BLINK_ERR_INVALID_ARGUMENT,
                "root " + std::to_string(root) + " out of range [0," + std::to_string(comm->nranks) + ")");
  if (count > (size_t(1) << 40))
    return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "count too large");
  if (comm->multiprocess && !comm->connected)
    return fail(comm, BLINK_ERR_INVALID_USAGE, "blink_connect has not been called");
  return BLINK_SUCCESS;
}

// Per-call tables that travel as kernel parameters (LaunchArgs).
void fill_param_tables(const Sized& s, LaunchArgs* a) {
  int acc = 0;
  for (size_t i = 0; i < s.htrees.size() && i < size_t(kMaxTrees); ++i) {
    a->ptrees[i] = s.htrees[i];
    acc += s.htrees[i].nchunks;
    a->tree_end[i] = acc;
  }
  a->merged_all = s.merged_all ? 1 : 0;
  a->mchunk = s.mchunk;
  a->mbytes = s.mbytes;
  if (s.merged_all) a->mtask = s.tasks[0];
}

// ---------------------------------------------------------------- LL protocol
constexpr size_t kLLOneLaunchMax = 64 << 10;

// Does this call take the low-latency protocol, and where are the one-hop
// slices?  The decision depends only on the call and the config, so every rank
// takes it alike.  AllReduce: the plan's m one-hop trees (tree j rooted at j,
// slice j = its split range, R#11).  Broadcast: the one-hop star.
bool ll_slices(blink_comm_t c, const Plan& plan, int coll, size_t count, int es,
               int64_t lo[kMaxRanks + 1]) {
  const int m = c->nranks;
  const size_t bytes = count * size_t(es);
  if (c->ll_bytes == 0 || m < 2 || bytes == 0 || bytes > c->cfg.ll_max_bytes || !plan.switch_model)
    return false;
  if (coll == kBroadcast) {
    lo[0] = 0;
    return plan.trees.size() == 1;
  }
  if (coll != kAllReduce || int(plan.trees.size()) != m) return false;
  auto key = std::make_pair(count, es);
  auto it = c->ll_lo.find(key);
  if (it == c->ll_lo.end()) {
    std::vector<TreeRange> rr;
    std::string err;
    if (size_plan(plan, count, es, c->cfg, 1, &rr, &err) != BLINK_SUCCESS || int(rr.size()) != m)
      return false;
    std::vector<int64_t> b(m + 1);
    for (int j = 0; j < m; ++j) {
      if (plan.trees[j].root != j || plan.trees[j].depth != 1) return false;
      if (j > 0 && rr[j].lo != rr[j - 1].hi) return false;
      b[j] = rr[j].lo * es;
    }
    b[m] = rr[m - 1].hi * es;
    if (b[0] != 0 || b[m] != int64_t(bytes)) return false;
    it = c->ll_lo.emplace(key, b).first;
  }
  for (int j = 0; j <= m; ++j) lo[j] = it->second[j];
  return true;
}

bool trace_on() {  // BLINK_TRACE (read per launch: tests toggle it at run time)
  return getenv("BLINK_TRACE") != nullptr;
}

bool link_graph(blink_comm_t c) { return !c->graph.switch_model && !c->graph.multi_server; }

// Small calls on a link graph's single minimum-depth tree (R#27) take the
// LL protocol too when every rank's whole buffer fits one LL slot
// (ll_tree_max: 128 KiB by default).
bool ll_tree(blink_comm_t c, const Plan& plan, int coll, size_t bytes) {
  const int m = c->nranks;
  if (c->ll_bytes == 0 || m < 3 || bytes == 0 || bytes > c->cfg.ll_max_bytes || plan.switch_model ||
      plan.trees.size() != 1 || (coll != kBroadcast && coll != kAllReduce))
    return false;
  static const bool off = getenv("BLINK_LL_TREE") && getenv("BLINK_LL_TREE")[0] == '0';
  if (off) return false;
  return bytes <= ll_tree_max(c->cfg.ll_max_bytes) &&
         bytes <= 8 * (ll_cap_lines(c->cfg.ll_max_bytes, m, link_graph(c)) - 8);
}

void set_ll_tree(const Plan& plan, LLArgs* a) {
  a->tree = 1;
  a->tree_root = plan.trees[0].root;
  for (int u = 0; u < a->nranks; ++u) a->parent[u] = int8_t(plan.trees[0].parent[u]);
}

// Everything but the per-rank buffers.  `share` = ranks whose launches share
// this device (their CTAs split the SMs).
void fill_ll_args(blink_comm_t c, int coll, int dtype, int op, int root, size_t bytes,
                  const int64_t lo[kMaxRanks + 1], uint64_t* ctrl, int* err, int share, LLArgs* a) {
  const int m = c->nranks;
  a->nranks = m;
  a->coll = coll;
  a->dtype = dtype;
  a->op = op;
  a->root = root;
  a->bytes = int64_t(bytes);
  a->cap = int64_t(ll_cap_lines(c->cfg.ll_max_bytes, m, link_graph(c)));
  for (int j = 0; j <= m; ++j) a->lo[j] = lo[j];
  const int64_t lines = (int64_t(bytes) + 7) / 8;
  const int want = int((lines + kLLThreads - 1) / kLLThreads);
  const int cap = std::max(1, c->sms / std::max(1, share));
  a->ctas_per_rank = std::max(1, std::min(want, cap));
  a->ctrl = ctrl;
  a->err = err;
  a->timeout_ns = uint64_t(c->cfg.timeout_s * 1e9);
}

// ---------------------------------------------------------------- single-process launch
// NEXT-1: which calls run in the switch (the same decision on every rank:
// it depends only on the call, never on a rank's pointers)
bool nvls_call(int coll, int op) { return coll == kBroadcast || (coll == kAllReduce && op == BLINK_SUM); }

// Fill the NVLS launch of rank v for bytes [off, off + cnt) of the call.
NvlsArgs nvls_args(blink_comm_t cv, int n, int v, int coll, int dtype, int root, const char* send, char* recv,
                   size_t off, size_t cnt, uint64_t* const* flags, uint64_t* ctrl, int* err) {
  NvlsArgs a{};
  a.nranks = n;
  a.rank = v;
  a.coll = coll;
  a.dtype = dtype;
  a.root = root;
  a.bytes = int64_t(cnt);
  a.send = send ? send + off : nullptr;
  a.recv = recv ? recv + off : nullptr;
  a.uc = reinterpret_cast<char*>(cv->nvls.uc_va);
  a.mc = reinterpret_cast<char*>(cv->nvls.mc_va);
  for (int u = 0; u < n; ++u) a.flags[u] = flags[u];
  a.ctrl = ctrl;
  a.err = err;
  a.timeout_ns = uint64_t(cv->cfg.timeout_s * 1e9);
  return a;
}

// single process, one rank per device: one NVLS launch per rank and piece
blink_result_t clique_nvls(Clique* q, size_t bytes) {
  const int n = q->nranks;
  blink_comm_t c0 = q->comms[0];
  uint64_t* flags[kMaxRanks];
  for (int u = 0; u < n; ++u) flags[u] = q->comms[u]->flags;
  const size_t P = c0->nvls.size;
  for (size_t off = 0; off < bytes; off += P) {
    const size_t cnt = std::min(P, bytes - off);
    for (const Clique::Group& grp : q->groups) {
      const int v = __builtin_ctzll(grp.mask);
      blink_comm_t cv = q->comms[v];
      DeviceGuard g(cv->device);
      NvlsArgs a = nvls_args(cv, n, v, q->coll, q->dtype, q->root, static_cast<const char*>(q->pending[v].send),
                             static_cast<char*>(q->pending[v].recv), off, cnt, flags, q->ctrl[grp.key],
                             q->err_dev[grp.key]);
      cudaError_t e = launch_nvls(a, cv->sms, q->pending[v].stream);
      if (e != cudaSuccess) return fail(cv, BLINK_ERR_CUDA, std::string("NVLS launch: ") + cudaGetErrorString(e));
      cv->stats.launches++;
      cv->stats.last_ctas = cv->sms;
      cv->stats.last_steal_channels = 0;
      cv->stats.last_chunks = 0;
      cv->stats.last_trees = n;
      cv->stats.last_chunk_bytes = int64_t(cnt);
    }
    q->launches++;
  }
  return BLINK_SUCCESS;
}

blink_result_t clique_launch(Clique* q) {
  const int n = q->nranks;
  const int es = esize_of(blink_dtype_t(q->dtype));
  const size_t bytes = q->count * es;
  q->calls++;
  blink_comm_t c0 = q->comms[0];
  if (n == 1) {
    DeviceGuard g(c0->device);
    CUDA_TRY(c0, launch_copy(q->pending[0].recv, q->coll == kBroadcast ? q->pending[0].send
                                                                       : q->pending[0].send,
                             bytes, q->pending[0].stream));
    q->launches++;
    return BLINK_SUCCESS;
  }
  const Plan* plan = nullptr;
  blink_result_t r = get_plan(c0, q->coll, q->root, bytes, &plan);
  if (r != BLINK_SUCCESS) return r;
  bool vec = true;
  for (int v = 0; v < n; ++v) {
    const Pending& p = q->pending[v];
    const bool reads_send = q->coll != kBroadcast || v == q->root;
    if (reads_send && !aligned16(p.send)) vec = false;
    if (!aligned16(p.recv)) vec = false;
  }
  if (is_block_coll(q->coll) && (bytes % kGrain) != 0) vec = false;  // block starts unaligned
  const bool all_one_launch = q->groups.size() == 1;
  // MIAD: the chunk size for this call from the previous calls'
  // measured throughput (single host thread decides for every rank)
  Clique::MiadRun* mr = nullptr;
  size_t chunk_override = 0;
  // one launch holding every rank has no handshake for LL to save; there it
  // pays only for Broadcast below kLLOneLaunchMax (A/B: scripts/per_rank_trace.py).
  // A one-launch AllReduce runs the merged channel on the register path
  // instead (scripts/ab_small.py, m = 8: 1 KiB 6.4 -> 4.1 us, 64 KiB 7.1 ->
  // 4.5 us; Broadcast stays on LL: 3.3 vs 4.3 us at 1 KiB)
  int64_t ll_lo[kMaxRanks + 1] = {};
  // the R#27 tree in LL: in one launch only up to kLLOneLaunchMax (128 KiB
  // ran 10-70% slower than the register path, e.g. DGX-1V AllReduce 15.0 vs
  // 12.5 us; 64 KiB mostly faster, 10.7 vs 12.4 us)
  const bool lltree = ll_tree(c0, *plan, q->coll, bytes) && (q->groups.size() > 1 || bytes <= kLLOneLaunchMax);
  const bool one_launch_ll = q->coll != kAllReduce && bytes <= kLLOneLaunchMax;
  const bool ll = lltree || ((q->groups.size() > 1 || one_launch_ll) &&
                             ll_slices(c0, *plan, q->coll, q->count, es, ll_lo));
  if (q->nvls && !ll && nvls_call(q->coll, q->op)) return clique_nvls(q, bytes);
  // MIAD does not step while a stream is being captured into a CUDA graph:
  // its event timing cannot run inside a capture
  bool capturing = false;
  for (int v = 0; v < n && !capturing; ++v) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(q->pending[v].stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
      capturing = true;
  }
  if (c0->cfg.autotune && !ll && capturing) {
    // freeze: a captured call takes the chunk the eager calls have tuned so
    // far (the static table's if none ran), without timing it
    auto mit = q->miad.find(std::make_tuple(q->coll, q->coll == kBroadcast ? q->root : -1, q->dtype, q->count));
    if (mit != q->miad.end()) chunk_override = mit->second.st.phase == 2 ? mit->second.st.best : mit->second.st.chunk;
  }
  if (c0->cfg.autotune && !ll && !capturing) {
    auto mk = std::make_tuple(q->coll, q->coll == kBroadcast ? q->root : -1, q->dtype, q->count);
    auto mit = q->miad.find(mk);
    if (mit == q->miad.end()) {
      // start from the static table's chunk ("a small value"; the
      // paper's 1 MB was for its hardware, R#15)
      std::vector<TreeRange> rr;
      std::string err;
      const int hint = std::max(1, co_resident_budget(c0, c0->device, q->dtype, q->op, q->coll) /
                                       std::max<int>(1, int(plan->trees.size())));
      size_t init = size_t(1) << 20;
      if (size_plan(*plan, q->count, es, c0->cfg, hint, &rr, &err) == BLINK_SUCCESS && !rr.empty())
        init = size_t(rr[0].chunk) * es;
      mit = q->miad.emplace(mk, Clique::MiadRun()).first;
      blink_miad_init(&mit->second.st, init, 16 << 10, size_t(64) << 20);
    }
    mr = &mit->second;
    if (mr->pending && cudaEventQuery(mr->ev1) == cudaSuccess) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, mr->ev0, mr->ev1);
      if (ms > 0.f) blink_miad_step(&mr->st, double(bytes) / (double(ms) * 1e-3));
      mr->pending = false;
    }
    chunk_override = mr->st.phase == 2 ? mr->st.best : mr->st.chunk;
    mr->calls++;
  }
  bool timed = false;
  // per-rank launches: fork every rank's launch stream off its stream before
  // any launch and join after all of them, so that ranks sharing one user
  // stream still run concurrently
  if (q->per_rank)
    for (int v = 0; v < n; ++v) {
      DeviceGuard g(q->comms[v]->device);
      CUDA_TRY(c0, cudaEventRecord(q->rfork[v], q->pending[v].stream));
      CUDA_TRY(c0, cudaStreamWaitEvent(q->rstream[v], q->rfork[v], 0));
    }
  if (ll) {  // low-latency protocol: one LL launch per group
    for (const Clique::Group& grp : q->groups) {
      LLArgs a{};
      int lead = -1;
      for (int v = 0; v < n; ++v)
        if ((grp.mask >> v) & 1) {
          if (lead < 0) lead = v;
          a.ranks[a.nlocal++] = int8_t(v);
        }
      blink_comm_t cd = q->comms[lead];
      DeviceGuard g(grp.device);
      int share = 0;
      for (const Clique::Group& g2 : q->groups)
        if (g2.device == grp.device) share += __builtin_popcountll(g2.mask);
      fill_ll_args(cd, q->coll, q->dtype, q->op, q->root, bytes, ll_lo, q->ctrl[grp.key],
                   q->err_dev[grp.key], share, &a);
      a.scope_sys = q->devices.size() > 1 ? 1 : 0;
      if (lltree) set_ll_tree(*plan, &a);
      for (int v = 0; v < n; ++v) {
        a.send[v] = static_cast<const char*>(q->pending[v].send);
        a.recv[v] = static_cast<char*>(q->pending[v].recv);
        a.ll[v] = reinterpret_cast<uint4*>(reinterpret_cast<char*>(q->comms[v]->flags) + kFlagBytes);
      }
      if (trace_on()) {
        uint64_t*& tb = q->trace[grp.key];
        if (!tb) CUDA_TRY(cd, cudaMalloc(&tb, sizeof(uint64_t) * kTraceSlots * 4096));
        a.trace = tb;
        q->trace_ctas[grp.key] = a.nlocal * a.ctas_per_rank;
      }
      cudaStream_t ls = q->per_rank ? q->rstream[lead] : q->pending[lead].stream;
      std::vector<cudaEvent_t> evs;
      for (int v = 0; v < n; ++v) {
        if (!((grp.mask >> v) & 1) || v == lead || q->pending[v].stream == ls) continue;
        cudaEvent_t e;
        CUDA_TRY(cd, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CUDA_TRY(cd, cudaEventRecord(e, q->pending[v].stream));
        CUDA_TRY(cd, cudaStreamWaitEvent(ls, e, 0));
        evs.push_back(e);
      }
      const int grid = a.nlocal * a.ctas_per_rank;
      cudaError_t le = launch_ll(a, grid, ls, use_coop() && !q->per_rank, use_pdl());
      if (le != cudaSuccess)
        return fail(cd, BLINK_ERR_CUDA, std::string("LL launch: ") + cudaGetErrorString(le));
      if (q->per_rank) CUDA_TRY(cd, cudaEventRecord(q->rjoin[lead], ls));
      q->launches++;
      for (int v = 0; v < n; ++v) {
        if (!((grp.mask >> v) & 1)) continue;
        q->comms[v]->stats.launches++;
        q->comms[v]->stats.last_ctas = grid;
        q->comms[v]->stats.last_steal_channels = 0;
        q->comms[v]->stats.last_chunks = 0;
        q->comms[v]->stats.last_trees = int(plan->trees.size());
        q->comms[v]->stats.last_chunk_bytes = 0;
      }
      if (!evs.empty()) {
        cudaEvent_t done;
        CUDA_TRY(cd, cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        CUDA_TRY(cd, cudaEventRecord(done, ls));
        for (int v = 0; v < n; ++v) {
          if (!((grp.mask >> v) & 1) || v == lead || q->pending[v].stream == ls) continue;
          CUDA_TRY(cd, cudaStreamWaitEvent(q->pending[v].stream, done, 0));
        }
        cudaEventDestroy(done);
        for (auto e : evs) cudaEventDestroy(e);
      }
    }
    if (q->per_rank)
      for (int v = 0; v < n; ++v) {
        DeviceGuard g(q->comms[v]->device);
        CUDA_TRY(c0, cudaStreamWaitEvent(q->pending[v].stream, q->rjoin[v], 0));
      }
    return BLINK_SUCCESS;
  }
  for (const Clique::Group& grp : q->groups) {
    const int dev = grp.device;
    const uint64_t mask = grp.mask;
    blink_comm_t cd = nullptr;
    for (int v = 0; v < n && !cd; ++v)
      if ((mask >> v) & 1) cd = q->comms[v];
    SizedKey key{q->coll, (q->coll == kBroadcast || q->coll == kGather) ? q->root : -1, q->dtype, q->count,
                 mask | (uint64_t(plan->trees.size()) << 32) |
                     (uint64_t(q->coll == kBroadcast && plan->trees.size() == 1) << 48),
                 chunk_override};
    auto it = q->sized.find(key);
    if (it == q->sized.end()) {
      Sized s;
      int budget = co_resident_budget(cd, dev, q->dtype, q->op, q->coll);
      // launch groups sharing a device run concurrently: split its CTAs
      int share = 0;
      for (const Clique::Group& g2 : q->groups) share += g2.device == dev;
      budget = std::max(1, budget / std::max(1, share));
      std::vector<uint64_t> gm;
      for (const Clique::Group& g2 : q->groups) gm.push_back(g2.mask);
      r = build_sized(cd, *plan, q->count, es, mask, gm, budget, &s, chunk_override);
      if (r != BLINK_SUCCESS) return r;
      r = finalize_tables(cd, dev, es, &s);
      if (r != BLINK_SUCCESS) return r;
      it = q->sized.emplace(key, std::move(s)).first;
    }
    Sized& s = it->second;
    LaunchArgs a{};
    a.tasks = s.d_tasks;
    a.trees = s.d_trees;
    a.ntrees = int(plan->trees.size());
    fill_param_tables(s, &a);
    a.nranks = n;
    a.coll = q->coll;
    a.dtype = q->dtype;
    a.op = q->op;
    a.exit_wait = all_one_launch ? 0 : 1;
    a.scope_sys = q->devices.size() > 1 ? 1 : 0;
    a.bcast_root = (q->coll == kBroadcast || q->coll == kGather) ? q->root : -1;
    a.use_tma = use_tma() && !s.lsu;
    a.smem_bytes = smem_bytes();
    a.tile_bytes = tile_bytes();
    a.store_depth = store_depth();
    a.split_ring = split_ring();
    a.copy_stages = copy_stages();
    a.chan0 = s.chan0;
    a.nchan = s.nchan;
    a.l2_hint = l2_hint();
    a.defer_signal = defer_signal();
    a.nctr = s.nctr;
    a.ctrl = q->ctrl[grp.key];
    if (trace_on()) {
      uint64_t*& tb = q->trace[grp.key];
      if (!tb) CUDA_TRY(cd, cudaMalloc(&tb, sizeof(uint64_t) * kTraceSlots * 4096));
      a.trace = tb;
      q->trace_ctas[grp.key] = s.ctas;
    }
    a.timeout_ns = uint64_t(cd->cfg.timeout_s * 1e9);
    a.err = q->err_dev[grp.key];
    for (int v = 0; v < n; ++v) {
      a.send[v] = const_cast<char*>(static_cast<const char*>(q->pending[v].send));
      a.recv[v] = static_cast<char*>(q->pending[v].recv);
      a.flags[v] = q->comms[v]->flags;
      if (q->coll == kGather && !a.recv[v]) {  // a relay on a link-graph Gather chain
        bool relay = false;
        for (const Tree& t : plan->trees) relay = relay || (t.parent[v] >= 0 && t.root != v);
        if (relay) {
          blink_comm* cv = q->comms[v];
          const size_t need = size_t(n) * bytes;
          if (cv->scratch_bytes < need) {
            DeviceGuard gv(cv->device);
            RelaxedCapture rc;
            if (cv->scratch) cudaFree(cv->scratch);
            cv->scratch = nullptr;
            cv->scratch_bytes = 0;
            CUDA_TRY(cd, cudaMalloc(&cv->scratch, need));
            cv->scratch_bytes = need;
          }
          a.recv[v] = cv->scratch;
        }
      }
      if (q->coll == kReduceScatter && !plan->switch_model) {
        // link-graph ReduceScatter: inner ranks relay partials of other
        // blocks through an m-block relay area (library scratch); each root
        // writes its own block straight into recv
        blink_comm* cv = q->comms[v];
        const size_t need = size_t(n) * bytes;
        if (cv->scratch_bytes < need) {
          DeviceGuard gv(cv->device);
          RelaxedCapture rc;
          if (cv->scratch) cudaFree(cv->scratch);
          cv->scratch = nullptr;
          cv->scratch_bytes = 0;
          CUDA_TRY(cd, cudaMalloc(&cv->scratch, need));
          cv->scratch_bytes = need;
        }
        a.relay[v] = cv->scratch;
      }
      // block collectives address rank v's short buffer through tree v's range
      if (q->coll == kReduceScatter) a.recv[v] -= size_t(v) * bytes;
      if ((q->coll == kAllGather || q->coll == kGather) && a.send[v]) a.send[v] -= size_t(v) * bytes;
    }
    DeviceGuard g(dev);
    // launch on the first rank's stream of this device after the others' streams
    int lead = -1;
    for (int v = 0; v < n; ++v)
      if ((mask >> v) & 1) {
        lead = v;
        break;
      }
    cudaStream_t ls = q->pending[lead].stream;
    if (q->per_rank) ls = q->rstream[lead];  // forked off the rank's stream above
    std::vector<cudaEvent_t> evs;
    for (int v = 0; v < n; ++v) {
      if (!((mask >> v) & 1) || v == lead || q->pending[v].stream == ls) continue;
      cudaEvent_t e;
      CUDA_TRY(cd, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CUDA_TRY(cd, cudaEventRecord(e, q->pending[v].stream));
      CUDA_TRY(cd, cudaStreamWaitEvent(ls, e, 0));
      evs.push_back(e);
    }
    const bool time_it = mr && !timed && !mr->pending && mr->st.phase != 2 && mr->calls > 1;
    if (time_it) {
      if (!mr->ev0) {
        CUDA_TRY(cd, cudaEventCreate(&mr->ev0));
        CUDA_TRY(cd, cudaEventCreate(&mr->ev1));
      }
      CUDA_TRY(cd, cudaEventRecord(mr->ev0, ls));
    }
    // per-rank launches rely on every group's grid fitting the device at once
    // (each takes 1/m of the co-resident CTAs); the cooperative attribute
    // cannot promise co-residency across launches
    cudaError_t le = launch_exec(a, s.ctas, cd->cfg.threads, vec, ls, use_coop() && !q->per_rank, use_pdl());
    if (le != cudaSuccess)
      return fail(cd, BLINK_ERR_CUDA, std::string("exec launch: ") + cudaGetErrorString(le));
    if (q->per_rank) CUDA_TRY(cd, cudaEventRecord(q->rjoin[lead], ls));
    if (time_it) {
      CUDA_TRY(cd, cudaEventRecord(mr->ev1, ls));
      mr->pending = true;
      timed = true;
    }
    q->launches++;
    for (int v = 0; v < n; ++v) {
      if (!((mask >> v) & 1)) continue;
      q->comms[v]->stats.launches++;
      q->comms[v]->stats.last_ctas = s.ctas;
      q->comms[v]->stats.last_steal_channels = s.nchan;
      q->comms[v]->stats.last_chunks = s.chunks;
      q->comms[v]->stats.last_trees = int(plan->trees.size());
      q->comms[v]->stats.last_chunk_bytes = s.ranges.empty() ? 0 : s.ranges[0].chunk * es;
    }
    if (!evs.empty()) {
      cudaEvent_t done;
      CUDA_TRY(cd, cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      CUDA_TRY(cd, cudaEventRecord(done, ls));
      for (int v = 0; v < n; ++v) {
        if (!((mask >> v) & 1) || v == lead || q->pending[v].stream == ls) continue;
        CUDA_TRY(cd, cudaStreamWaitEvent(q->pending[v].stream, done, 0));
      }
      cudaEventDestroy(done);
      for (auto e : evs) cudaEventDestroy(e);
    }
  }
  if (q->per_rank)
    for (int v = 0; v < n; ++v) {
      DeviceGuard g(q->comms[v]->device);
      CUDA_TRY(c0, cudaStreamWaitEvent(q->pending[v].stream, q->rjoin[v], 0));
    }
  return BLINK_SUCCESS;
}

blink_result_t clique_post(blink_comm_t comm, int coll, const void* send, void* recv, size_t count,
                           blink_dtype_t dtype, int op, int root, void* stream) {
  Clique* q = comm->clique;
  std::lock_guard<std::mutex> lk(q->mu);
  for (auto& kv : q->err_host)
    if (*kv.second != 0) {
      if (getenv("BLINK_DUMP_FLAGS")) {  // debugging aid: the flag words of chunk 0 of every tree
        cudaDeviceSynchronize();
        for (int v = 0; v < q->nranks; ++v) {
          std::vector<uint64_t> w(kFlagWords);
          cudaMemcpy(w.data(), q->comms[v]->flags, kFlagBytes, cudaMemcpyDeviceToHost);
          fprintf(stderr, "[blink] rank %d entry:", v);
          for (int u = 0; u < q->nranks; ++u) fprintf(stderr, " %llu", (unsigned long long)w[entry_idx(u)]);
          fprintf(stderr, "  bflag[t][0]:");
          for (int t = 0; t < q->nranks; ++t) fprintf(stderr, " %llu", (unsigned long long)w[bflag_idx(t, 0)]);
          fprintf(stderr, "  pflag[t][child][0]:");
          for (int t = 0; t < q->nranks; ++t)
            for (int u = 0; u < q->nranks; ++u)
              if (w[pflag_idx(t, u, 0)]) fprintf(stderr, " t%d/c%d=%llu", t, u, (unsigned long long)w[pflag_idx(t, u, 0)]);
          fprintf(stderr, "\n");
        }
      }
      return fail(comm, blink_result_t(*kv.second),
                  "a previous launch aborted (flag wait timed out in launch group " +
                      std::to_string(kv.first) + ")");
    }
  if (q->nposted == 0) {
    q->coll = coll;
    q->root = root;
    q->dtype = dtype;
    q->op = op;
    q->count = count;
  } else if (q->coll != coll || q->count != count || q->dtype != int(dtype) ||
             (!is_push_coll(coll) && q->op != op) ||
             ((coll == kBroadcast || coll == kGather) && q->root != root)) {
    return fail(comm, BLINK_ERR_INVALID_USAGE,
                "rank " + std::to_string(comm->rank) +
                    " called a different collective/count/dtype/op/root than the ranks already "
                    "posted in this batch");
  }
  Pending& p = q->pending[comm->rank];
  if (p.posted)
    return fail(comm, BLINK_ERR_INVALID_USAGE,
                "rank " + std::to_string(comm->rank) + " posted twice before all ranks called");
  p.posted = true;
  p.send = send;
  p.recv = recv;
  p.stream = static_cast<cudaStream_t>(stream);
  if (++q->nposted < q->nranks) return BLINK_SUCCESS;
  blink_result_t r = BLINK_SUCCESS;
  if (count > 0) r = clique_launch(q);
  if (r != BLINK_SUCCESS) comm->last_error = g_last_error;
  for (auto& pp : q->pending) pp = Pending();
  q->nposted = 0;
  return r;
}

// ---------------------------------------------------------------- multi-process
struct Blob {
  char magic[8];
  int32_t rank, nranks, device, pid;
  char bus_id[32];
  cudaIpcMemHandle_t flags_h;
  cudaIpcMemHandle_t staging_h;
  uint64_t staging_bytes;
  uint64_t ll_bytes;
  uint64_t ll_max_bytes;  // the LL-or-tree decision must be the same on every rank
  uint64_t shallow_max_bytes;       // so must the plan choices by size (R#27,
  uint64_t onehop_bcast_max_bytes;  // the switch Broadcast star)
  uint64_t chunk_fp;                // and every input of the chunk table (a chunk's flags name bytes)
  int32_t nvls_offer, pad2;         // rank 0: a multicast object for NEXT-1 (NvlsShare: FABRIC handle or POSIX fd below)
  uint64_t nvls_size;
  unsigned char nvls_handle[64];
};

// Fingerprint of everything the chunk table (size_plan / build_sized) reads:
// config fields, the SM count and the environment overrides.  Ranks whose
// chunking differs would consume each other's flags for different byte
// ranges, so blink_connect refuses to mix them.
uint64_t chunking_fingerprint(blink_comm_t comm) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= (v >> (8 * i)) & 0xffu;
      h *= 1099511628211ull;
    }
  };
  mix(comm->cfg.chunk_bytes);
  mix(uint64_t(comm->cfg.ctas));
  mix(uint64_t(comm->cfg.threads));
  mix(uint64_t(comm->cfg.autotune));
  mix(uint64_t(comm->cfg.nvls));
  mix(uint64_t(comm->cfg.nvls_bytes));
  uint64_t d;
  memcpy(&d, &comm->cfg.mwu_eps, sizeof d);  // the plan's trees (MWU / ILP settings)
  mix(d);
  memcpy(&d, &comm->cfg.ilp_gap, sizeof d);
  mix(d);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, comm->device);
  mix(uint64_t(sms));
  static const char* envs[] = {"BLINK_CHUNK_BYTES", "BLINK_CTAS", "BLINK_MIN_CHUNK", "BLINK_MIN_CHUNK_DEEP",
                               "BLINK_DEEP_CAP", "BLINK_CHUNKS_PER_CTA", "BLINK_SMEM_KB", "BLINK_TILE",
                               "BLINK_TMA", "BLINK_ONE_CHUNK", "BLINK_MERGE", "BLINK_DYNAMIC",
                               "BLINK_PACK", "BLINK_THREADS", "BLINK_MIAD", "BLINK_ILP_DIVES",
                               "BLINK_LL_TREE", "BLINK_ALLOC"};
  for (const char* name : envs) {
    const char* e = getenv(name);
    mix(0x5eedull);
    for (const char* q = e ? e : ""; *q; ++q) mix(uint64_t(uint8_t(*q)));
  }
  return h;
}
constexpr int kMaxVmmChunks = 128;
struct RegBlob {
  char magic[8];
  int32_t rank, kind;              // kind 0: cudaMalloc memory (legacy IPC handle)
  cudaIpcMemHandle_t h;            // kind 1: VMM chunks (PyTorch expandable segments)
  uint64_t offset, bytes;
  int32_t pid, nchunks;            // kind 1: exporter pid and its POSIX fds, one per chunk
  struct {
    int64_t off;
    uint64_t size;
    int32_t fd, pad;
  } chunks[kMaxVmmChunks];
};

blink_result_t open_handle(blink_comm_t comm, const cudaIpcMemHandle_t& h, char** out) {
  std::string key(reinterpret_cast<const char*>(&h), sizeof h);
  auto it = comm->opened.find(key);
  if (it != comm->opened.end()) {
    *out = it->second;
    return BLINK_SUCCESS;
  }
  void* p = nullptr;
  CUDA_TRY(comm, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  comm->opened[key] = static_cast<char*>(p);
  *out = static_cast<char*>(p);
  return BLINK_SUCCESS;
}

bool resolve(blink_comm_t comm, const void* ptr, size_t bytes, char* out[kMaxRanks]) {
  const char* p = static_cast<const char*>(ptr);
  for (const Reg& r : comm->regs) {
    if (p >= r.buf && p + bytes <= r.buf + r.bytes) {
      size_t off = size_t(p - r.buf);
      for (int u = 0; u < comm->nranks; ++u) out[u] = r.peer[u] + off;
      return true;
    }
  }
  return false;
}

// MIAD across processes (NEXT-2).  Every rank makes the same
// sequence of autotuned calls, numbered by comm->miad_seq.  Rank 0 runs the
// MIAD controller on its own CUDA-event time of the previous call (its kernel
// waits for every peer through the flags, so that time is the collective's,
// i.e. the slowest rank's) and publishes call s's chunk size in its flag
// words, slot s % kMiadSlots, with a stream-ordered store before its launch.
// Every other rank reads that slot (through its IPC mapping of rank 0's flags)
// until the slot carries tag s + 1: all ranks chunk call s identically.  Once
// rank 0 publishes a converged size (phase 2), both sides stop for that key.
// Slot reuse is safe: rank 0 overwrites slot s at call s + kMiadSlots, after
// its kernel for call s + kMiadSlots - 1, which needs every rank's entry for
// that call -- so every reader has long read slot s.
blink_result_t mp_miad_chunk(blink_comm_t comm, int coll, int root, blink_dtype_t dtype, size_t count,
                             const Plan& plan, cudaStream_t stream, size_t* chunk,
                             blink_comm::MpMiad** out) {
  const auto key = std::make_tuple(coll, coll == kBroadcast ? root : -1, int(dtype), count);
  blink_comm::MpMiad& m = comm->mp_miad[key];
  *out = &m;
  if (m.done) {
    *chunk = m.chunk;
    return BLINK_SUCCESS;
  }
  const uint64_t seq = comm->miad_seq++;
  const int es = esize_of(dtype);
  size_t c = 0;
  bool conv = false;
  if (comm->rank == 0) {
    if (m.calls == 0) {  // start from the static table's chunk (R#15)
      std::vector<TreeRange> rr;
      std::string err;
      const int hint = std::max(1, co_resident_budget(comm, comm->device, dtype, BLINK_SUM, coll) /
                                       std::max<int>(1, int(plan.trees.size())));
      size_t init = size_t(1) << 20;
      if (size_plan(plan, count, es, comm->cfg, hint, &rr, &err) == BLINK_SUCCESS && !rr.empty())
        init = size_t(rr[0].chunk) * es;
      blink_miad_init(&m.st, init, 16 << 10, size_t(64) << 20);
      CUDA_TRY(comm, cudaEventCreate(&m.ev0));
      CUDA_TRY(comm, cudaEventCreate(&m.ev1));
    } else if (m.pending && cudaEventQuery(m.ev1) == cudaSuccess) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, m.ev0, m.ev1);
      if (ms > 0.f) blink_miad_step(&m.st, double(count * es) / (double(ms) * 1e-3));
      m.pending = false;
    }
    conv = m.st.phase == 2;
    c = conv ? m.st.best : m.st.chunk;
    cudaError_t e = launch_store2(comm->flags + miad_idx(seq), seq + 1, uint64_t(c) | (uint64_t(conv) << 56),
                                  stream);
    if (e != cudaSuccess) return fail(comm, BLINK_ERR_CUDA, std::string("MIAD publish: ") + cudaGetErrorString(e));
  } else {
    if (!comm->miad_stream) CUDA_TRY(comm, cudaStreamCreateWithFlags(&comm->miad_stream, cudaStreamNonBlocking));
    const uint64_t* src = comm->peer_flags[0] + miad_idx(seq);
    uint64_t v[2] = {0, 0};
    const auto t0 = std::chrono::steady_clock::now();
    for (int pass = 0;; ++pass) {
      CUDA_TRY(comm, cudaMemcpyAsync(v, src, sizeof v, cudaMemcpyDeviceToHost, comm->miad_stream));
      CUDA_TRY(comm, cudaStreamSynchronize(comm->miad_stream));
      if (v[0] == seq + 1) break;
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > comm->cfg.timeout_s)
        return fail(comm, BLINK_ERR_TIMEOUT,
                    "MIAD: rank 0 did not publish the chunk size of autotuned call " + std::to_string(seq));
      if (pass > 8) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    // the tag is stored after the value (with a fence): read the value again
    CUDA_TRY(comm, cudaMemcpyAsync(v, src, sizeof v, cudaMemcpyDeviceToHost, comm->miad_stream));
    CUDA_TRY(comm, cudaStreamSynchronize(comm->miad_stream));
    c = size_t(v[1] & ((uint64_t(1) << 56) - 1));
    conv = (v[1] >> 56) != 0;
  }
  m.done = conv;
  m.chunk = c;  // the last chunk every rank used for this key (also a capture's)
  m.calls++;
  *chunk = c;
  return BLINK_SUCCESS;
}

blink_result_t mp_run(blink_comm_t comm, int coll, char* send[kMaxRanks], char* recv[kMaxRanks],
                      size_t count, blink_dtype_t dtype, int op, int root, cudaStream_t stream,
                      char* const* relay = nullptr) {
  const int n = comm->nranks;
  const int es = esize_of(dtype);
  const size_t bytes = count * es;
  comm->calls++;
  const Plan* plan = nullptr;
  blink_result_t r = get_plan(comm, coll, root, bytes, &plan);
  if (r != BLINK_SUCCESS) return r;
  uint64_t mask = uint64_t(1) << comm->rank;
  size_t chunk_override = 0;
  blink_comm::MpMiad* mm = nullptr;
  cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
  const bool capturing = cudaStreamIsCapturing(stream, &cap_st) == cudaSuccess &&
                         cap_st != cudaStreamCaptureStatusNone;
  if (comm->cfg.autotune && capturing && (coll == kBroadcast || coll == kAllReduce)) {
    // a captured call neither times nor reads a slot: it takes the chunk of
    // the last eager autotuned call, which every rank used (static if none)
    auto mit = comm->mp_miad.find(std::make_tuple(coll, coll == kBroadcast ? root : -1, int(dtype), count));
    if (mit != comm->mp_miad.end()) chunk_override = mit->second.chunk;
  }
  if (comm->cfg.autotune && !capturing && (coll == kBroadcast || coll == kAllReduce)) {
    r = mp_miad_chunk(comm, coll, root, dtype, count, *plan, stream, &chunk_override, &mm);
    if (r != BLINK_SUCCESS) return r;
  }
  SizedKey key{coll, (coll == kBroadcast || coll == kGather) ? root : -1, int(dtype), count,
               mask | (uint64_t(plan->trees.size()) << 32), chunk_override};
  auto it = comm->sized.find(key);
  if (it == comm->sized.end()) {
    Sized s;
    int budget = co_resident_budget(comm, comm->device, dtype, op, coll);
    std::vector<uint64_t> gm;  // one group per process
    for (int u = 0; u < n; ++u) gm.push_back(uint64_t(1) << u);
    r = build_sized(comm, *plan, count, es, mask, gm, budget, &s, chunk_override);
    if (r != BLINK_SUCCESS) return r;
    r = finalize_tables(comm, comm->device, es, &s);
    if (r != BLINK_SUCCESS) return r;
    it = comm->sized.emplace(key, std::move(s)).first;
  }
  Sized& s = it->second;
  bool vec = true;
  for (int u = 0; u < n; ++u) {
    if (!aligned16(send[u]) || !aligned16(recv[u])) vec = false;  // (NULLs are aligned)
  }
  if (is_block_coll(coll) && (bytes % kGrain) != 0) vec = false;
  LaunchArgs a{};
  a.tasks = s.d_tasks;
  a.trees = s.d_trees;
  a.ntrees = int(plan->trees.size());
  fill_param_tables(s, &a);
  a.nranks = n;
  a.coll = coll;
  a.dtype = dtype;
  a.op = op;
  a.exit_wait = 1;
  a.scope_sys = 1;
  a.bcast_root = (coll == kBroadcast || coll == kGather) ? root : -1;
  a.use_tma = use_tma() && !s.lsu;
  a.smem_bytes = smem_bytes();
  a.tile_bytes = tile_bytes();
  a.store_depth = store_depth();
    a.split_ring = split_ring();
    a.copy_stages = copy_stages();
    a.chan0 = s.chan0;
    a.nchan = s.nchan;
  a.l2_hint = l2_hint();
  a.defer_signal = defer_signal();
  a.nctr = s.nctr;
  a.ctrl = comm->ctrl;
  a.timeout_ns = uint64_t(comm->cfg.timeout_s * 1e9);
  a.err = comm->err_dev;
  for (int u = 0; u < n; ++u) {
    a.send[u] = send[u];
    a.recv[u] = recv[u];
    a.flags[u] = comm->peer_flags[u];
    if (coll == kReduceScatter && a.recv[u]) a.recv[u] -= size_t(u) * bytes;
    if (relay) a.relay[u] = relay[u];
    if ((coll == kAllGather || coll == kGather) && a.send[u]) a.send[u] -= size_t(u) * bytes;
  }
  const bool time_it = mm && mm->ev0 && !mm->pending && !mm->done;  // rank 0 only
  if (time_it) CUDA_TRY(comm, cudaEventRecord(mm->ev0, stream));
  cudaError_t le = launch_exec(a, s.ctas, comm->cfg.threads, vec, stream, use_coop(), use_pdl());
  if (le != cudaSuccess)
    return fail(comm, BLINK_ERR_CUDA, std::string("exec launch: ") + cudaGetErrorString(le));
  if (time_it) {
    CUDA_TRY(comm, cudaEventRecord(mm->ev1, stream));
    mm->pending = true;
  }
  comm->stats.launches++;
  comm->stats.last_ctas = s.ctas;
  comm->stats.last_steal_channels = s.nchan;
  comm->stats.last_chunks = s.chunks;
  comm->stats.last_trees = int(plan->trees.size());
  comm->stats.last_chunk_bytes = s.ranges.empty() ? 0 : s.ranges[0].chunk * es;
  return BLINK_SUCCESS;
}

// ReduceScatter / AllGather across processes.  RS: peers read this rank's
// send (register it or it is staged), only the own recv is written.  AG: peers
// write this rank's recv (register it or it is staged), only the own send is
// read.  Staged calls run in pieces of P elements per block.
blink_result_t mp_block_collective(blink_comm_t comm, int coll, const void* sendbuf, void* recvbuf,
                                   size_t count, blink_dtype_t dtype, int op, int root,
                                   cudaStream_t stream) {
  const int m = comm->nranks, me = comm->rank;
  const int es = esize_of(dtype);
  const char* sb = static_cast<const char*>(sendbuf);
  char* rb = static_cast<char*>(recvbuf);
  char* sp[kMaxRanks] = {};
  char* rp[kMaxRanks] = {};
  if (coll == kReduceScatter && !comm->graph.switch_model) {
    // link graphs: inner ranks relay partials of other blocks, so every rank
    // needs a symmetric m-block relay area: the staging buffer's second half
    // (the first half holds the send blocks).  Pieces of P elements per block.
    const size_t P = std::max<size_t>(1, comm->staging_bytes / (2 * size_t(m) * es));
    const size_t half = P * size_t(m) * es;
    char* s2[kMaxRanks];
    char* rl[kMaxRanks];
    for (int u = 0; u < m; ++u) {
      s2[u] = comm->peer_staging[u];
      rl[u] = comm->peer_staging[u] + half;
    }
    for (size_t k0 = 0; k0 < count; k0 += P) {
      const size_t cnt = std::min(P, count - k0);
      for (int j = 0; j < m; ++j)
        CUDA_TRY(comm, launch_copy(comm->staging + size_t(j) * cnt * es, sb + (size_t(j) * count + k0) * es,
                                   cnt * es, stream));
      char* r2[kMaxRanks] = {};
      r2[me] = rb + k0 * es;  // only the root writes its recv: a local pointer suffices
      blink_result_t r = mp_run(comm, coll, s2, r2, cnt, dtype, op, -1, stream, rl);
      if (r != BLINK_SUCCESS) return r;
    }
    return BLINK_SUCCESS;
  }
  if (coll == kReduceScatter) {
    rp[me] = rb;
    if (resolve(comm, sendbuf, size_t(m) * count * es, sp))
      return mp_run(comm, coll, sp, rp, count, dtype, op, -1, stream);
  } else {
    sp[me] = const_cast<char*>(sb);
    // Every rank must take the same path (the flags name the same bytes).
    // Gather's non-roots may pass recvbuf = NULL, so Gather always stages;
    // AllGather's registration is collective (symmetric on every rank).
    if (coll == kAllGather && recvbuf && resolve(comm, recvbuf, size_t(m) * count * es, rp))
      return mp_run(comm, coll, sp, rp, count, dtype, op, root, stream);
  }
  const size_t P = std::max<size_t>(1, comm->staging_bytes / (size_t(m) * es));
  char* st[kMaxRanks];
  for (int u = 0; u < m; ++u) st[u] = comm->peer_staging[u];
  for (size_t k0 = 0; k0 < count; k0 += P) {
    const size_t cnt = std::min(P, count - k0);
    char* s2[kMaxRanks] = {};
    char* r2[kMaxRanks] = {};
    blink_result_t r;
    if (coll == kReduceScatter) {
      for (int j = 0; j < m; ++j)
        CUDA_TRY(comm, launch_copy(comm->staging + size_t(j) * cnt * es,
                                   sb + (size_t(j) * count + k0) * es, cnt * es, stream));
      r2[me] = rb + k0 * es;
      r = mp_run(comm, coll, st, r2, cnt, dtype, op, -1, stream);
      if (r != BLINK_SUCCESS) return r;
    } else {
      CUDA_TRY(comm, launch_copy(comm->staging + size_t(me) * cnt * es, sb + k0 * es, cnt * es, stream));
      s2[me] = comm->staging + size_t(me) * cnt * es;
      r = mp_run(comm, coll, s2, st, cnt, dtype, op, root, stream);
      if (r != BLINK_SUCCESS) return r;
      if (coll == kAllGather || me == root)
        for (int j = 0; j < m; ++j)
          CUDA_TRY(comm, launch_copy(rb + (size_t(j) * count + k0) * es,
                                     comm->staging + size_t(j) * cnt * es, cnt * es, stream));
    }
  }
  return BLINK_SUCCESS;
}

blink_result_t mp_collective(blink_comm_t comm, int coll, const void* sendbuf, void* recvbuf,
                             size_t count, blink_dtype_t dtype, int op, int root, void* stream_) {
  if (*comm->err_host != 0)
    return fail(comm, blink_result_t(*comm->err_host),
                "a previous launch aborted (flag wait timed out)");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int es = esize_of(dtype);
  const size_t bytes = count * es;
  DeviceGuard g(comm->device);
  if (comm->nranks == 1) {
    CUDA_TRY(comm, launch_copy(recvbuf, sendbuf, bytes, stream));
    comm->stats.launches++;
    return BLINK_SUCCESS;
  }
  if (is_block_coll(coll))
    return mp_block_collective(comm, coll, sendbuf, recvbuf, count, dtype, op, root, stream);
  {  // low-latency protocol: user buffers are only touched by their own rank
    const Plan* plan = nullptr;
    blink_result_t r = get_plan(comm, coll, root, bytes, &plan);
    if (r != BLINK_SUCCESS) return r;
    int64_t lo[kMaxRanks + 1] = {};
    const bool lltree = ll_tree(comm, *plan, coll, bytes);
    if (lltree || ll_slices(comm, *plan, coll, count, es, lo)) {
      comm->calls++;
      LLArgs a{};
      a.ranks[a.nlocal++] = int8_t(comm->rank);
      fill_ll_args(comm, coll, dtype, op, root, bytes, lo, comm->ctrl, comm->err_dev, 1, &a);
      a.scope_sys = 1;
      if (lltree) set_ll_tree(*plan, &a);
      a.send[comm->rank] = static_cast<const char*>(sendbuf);
      a.recv[comm->rank] = static_cast<char*>(recvbuf);
      for (int u = 0; u < comm->nranks; ++u)
        a.ll[u] = reinterpret_cast<uint4*>(reinterpret_cast<char*>(comm->peer_flags[u]) + kFlagBytes);
      cudaError_t le = launch_ll(a, a.ctas_per_rank, stream, false, use_pdl());
      if (le != cudaSuccess)
        return fail(comm, BLINK_ERR_CUDA, std::string("LL launch: ") + cudaGetErrorString(le));
      comm->stats.launches++;
      comm->stats.last_ctas = a.ctas_per_rank;
      comm->stats.last_steal_channels = 0;
      comm->stats.last_chunks = 0;
      comm->stats.last_trees = int(plan->trees.size());
      comm->stats.last_chunk_bytes = 0;
      return BLINK_SUCCESS;
    }
  }
  if (comm->nvls_on && nvls_call(coll, op)) {  // NEXT-1: the one-hop trees in the switch
    const size_t P = comm->nvls.size;
    for (size_t off = 0; off < bytes; off += P) {
      const size_t cnt = std::min(P, bytes - off);
      NvlsArgs a = nvls_args(comm, comm->nranks, comm->rank, coll, dtype, root,
                             static_cast<const char*>(sendbuf), static_cast<char*>(recvbuf), off, cnt,
                             comm->peer_flags, comm->ctrl, comm->err_dev);
      comm->calls++;
      cudaError_t e = launch_nvls(a, comm->sms, stream);
      if (e != cudaSuccess) return fail(comm, BLINK_ERR_CUDA, std::string("NVLS launch: ") + cudaGetErrorString(e));
      comm->stats.launches++;
      comm->stats.last_ctas = comm->sms;
      comm->stats.last_steal_channels = 0;
      comm->stats.last_chunks = 0;
      comm->stats.last_trees = comm->nranks;
      comm->stats.last_chunk_bytes = int64_t(cnt);
    }
    return BLINK_SUCCESS;
  }
  char* sp[kMaxRanks] = {};
  char* rp[kMaxRanks] = {};
  const bool recv_ok = resolve(comm, recvbuf, bytes, rp);
  if (coll == kBroadcast) {
    // only the root reads a send buffer, its own: no registration needed
    if (comm->rank == root) sp[root] = const_cast<char*>(static_cast<const char*>(sendbuf));
    if (recv_ok) return mp_run(comm, coll, sp, rp, count, dtype, op, root, stream);
  } else if (recv_ok && resolve(comm, sendbuf, bytes, sp)) {
    // zero-copy: registered symmetric buffers (parents pull from leaves' send)
    return mp_run(comm, coll, sp, rp, count, dtype, op, root, stream);
  }
  // staging path: in-place collective on the symmetric staging buffer, in pieces
  const size_t piece_elems = comm->staging_bytes / es;
  for (size_t off = 0; off < count; off += piece_elems) {
    size_t cnt = std::min(piece_elems, count - off);
    const char* s = static_cast<const char*>(sendbuf) + off * es;
    char* d = static_cast<char*>(recvbuf) + off * es;
    if (coll == kAllReduce || comm->rank == root)
      CUDA_TRY(comm, launch_copy(comm->staging, s, cnt * es, stream));
    char* st[kMaxRanks];
    for (int u = 0; u < comm->nranks; ++u) st[u] = comm->peer_staging[u];
    blink_result_t r = mp_run(comm, coll, st, st, cnt, dtype, op, root, stream);
    if (r != BLINK_SUCCESS) return r;
    CUDA_TRY(comm, launch_copy(d, comm->staging, cnt * es, stream));
  }
  return BLINK_SUCCESS;
}

}  // namespace

// =============================================================== C ABI
extern "C" {

void blink_config_default(blink_config_t* c) {
  if (!c) return;
  c->mwu_eps = 0.1;
  c->ilp_gap = 0.05;
  c->chunk_bytes = 0;
  c->ctas = 0;
  c->threads = 256;
  c->timeout_s = 30.0;
  c->onehop_bcast_max_bytes = 256 << 10;
  c->staging_bytes = 64 << 20;
  c->autotune = 0;
  c->launch_per_rank = 0;
  c->ll_max_bytes = 256 << 10;
  c->shallow_max_bytes = 256 << 10;
  c->nvls = 0;
  c->nvls_bytes = size_t(64) << 20;
}

void blink_miad_init(blink_miad_t* st, size_t init, size_t min_chunk, size_t max_chunk) {
  if (!st) return;
  memset(st, 0, sizeof *st);
  st->min_chunk = std::max<size_t>(kGrain, min_chunk);
  st->max_chunk = std::max(st->min_chunk, max_chunk);
  st->init = std::min(std::max(init, st->min_chunk), st->max_chunk);
  st->step = st->init;
  st->chunk = st->init;
  st->best = st->init;
  st->tol = 0.01;
}

size_t blink_miad_step(blink_miad_t* st, double thr) {
  if (!st) return 0;
  st->iters++;
  const bool first = st->iters == 1;
  if (first || thr > st->best_thr) {
    st->best_thr = thr;
    st->best = st->chunk;
  }
  const bool increasing = first || thr > st->last_thr * (1.0 + st->tol);
  st->last_thr = thr;
  if (st->phase == 0) {                  // multiplicative increase
    if (increasing && st->chunk * 2 <= st->max_chunk) {
      st->chunk *= 2;
    } else if (increasing) {             // hit the ceiling while still improving
      st->phase = 2;
      st->chunk = st->best;
    } else {                             // throughput dropped: additive decrease
      st->phase = 1;
      st->chunk = st->chunk > st->step + st->min_chunk ? st->chunk - st->step : st->best;
      if (st->chunk == st->best) st->phase = 2;
    }
  } else if (st->phase == 1) {           // additive decrease while it helps
    if (increasing && st->chunk > st->step + st->min_chunk) {
      st->chunk -= st->step;
    } else {
      st->phase = 2;
      st->chunk = st->best;
    }
  } else {
    st->chunk = st->best;
  }
  st->chunk = (st->chunk + kGrain - 1) / kGrain * kGrain;
  return st->chunk;
}

const char* blink_result_string(blink_result_t r) {
  switch (r) {
    case BLINK_SUCCESS: return "success";
    case BLINK_ERR_CUDA: return "CUDA error";
    case BLINK_ERR_SYSTEM: return "system error";
    case BLINK_ERR_INTERNAL: return "internal error";
    case BLINK_ERR_INVALID_ARGUMENT: return "invalid argument";
    case BLINK_ERR_INVALID_USAGE: return "invalid usage";
    case BLINK_ERR_TOPOLOGY: return "topology error";
    case BLINK_ERR_UNSUPPORTED: return "unsupported";
    case BLINK_ERR_TIMEOUT: return "timeout";
  }
  return "unknown";
}

const char* blink_last_error(blink_comm_t comm) {
  return comm ? comm->last_error.c_str() : g_last_error.c_str();
}

blink_result_t blink_plan_json(const blink_graph_t* graph, int nranks, const blink_config_t* cfg_in,
                               int is_allreduce, int root, size_t count, blink_dtype_t dtype,
                               char* json, size_t* json_bytes) {
  if (!json_bytes) return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "json_bytes is NULL");
  if (nranks < 1 || nranks > kMaxRanks)
    return fail(nullptr, BLINK_ERR_UNSUPPORTED, "nranks out of range");
  int es = esize_of(dtype);
  if (!es) return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "bad dtype");
  blink_config_t cfg = resolve_cfg(cfg_in);
  Graph g;
  std::string err;
  blink_result_t r = build_graph(graph, nranks, &g, &err);
  if (r != BLINK_SUCCESS) return fail(nullptr, r, err);
  Plan p;
  // is_allreduce: 0 Broadcast, 1 AllReduce, 2 ReduceScatter, 3 AllGather, 4 Gather
  if (is_allreduce < 0 || is_allreduce > kGather)
    return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "collective code must be 0..4");
  const int coll = is_allreduce;
  if (is_block_coll(coll) && g.multi_server) {
    r = BLINK_ERR_UNSUPPORTED;
    err = "multi-server graphs support AllReduce only";
  } else if (is_block_coll(coll) && !g.switch_model) {
    r = make_block_plan(g, coll, root, &p, &err);
  } else if (is_block_coll(coll)) {  // one-hop stars, tree j owns block j (as get_plan)
    r = make_plan(g, kAllReduce, root, cfg, &p, &err);
    p.coll = coll;
    p.blocks = true;
    if (coll == kGather)
      for (Tree& t : p.trees)
        for (int v = 0; v < int(t.parent.size()); ++v)
          if (t.parent[v] >= 0 && v != root) t.parent[v] = -2;
  } else if (use_shallow_plan(g, coll, count * size_t(es), cfg)) {
    r = make_shallow_plan(g, coll, root, &p, &err);
  } else {
    r = make_plan(g, coll, root, cfg, &p, &err);
  }
  if (r != BLINK_SUCCESS) return fail(nullptr, r, err);
  std::vector<TreeRange> ranges;
  int hint = std::max(1, (cfg.ctas > 0 ? cfg.ctas : 296) / int(p.trees.size()));
  r = size_plan(p, count, es, cfg, hint, &ranges, &err);
  if (r != BLINK_SUCCESS) return fail(nullptr, r, err);
  std::string s = plan_to_json(p, count, es, ranges, 0);
  size_t need = s.size() + 1;
  size_t cap = *json_bytes;
  *json_bytes = need;
  if (!json || cap < need) return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "json buffer too small");
  memcpy(json, s.c_str(), need);
  return BLINK_SUCCESS;
}

blink_result_t blink_topology_json(int ndev, const char* const* bus_ids, char* json, size_t* json_bytes) {
  if (!json_bytes || (ndev > 0 && !bus_ids)) return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "NULL argument");
  if (ndev < 1 || ndev > kMaxRanks) return fail(nullptr, BLINK_ERR_UNSUPPORTED, "ndev out of range");
  std::vector<std::string> bus;
  for (int i = 0; i < ndev; ++i) {
    if (!bus_ids[i]) return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "NULL bus id");
    bus.push_back(bus_ids[i]);
  }
  Probe p;
  std::string err;
  blink_result_t r = probe_topology(bus, &p, &err);
  if (r != BLINK_SUCCESS) return fail(nullptr, r, err);
  std::string s = probe_to_json(p);
  const size_t need = s.size() + 1, cap = *json_bytes;
  *json_bytes = need;
  if (!json || cap < need) return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "json buffer too small");
  memcpy(json, s.c_str(), need);
  return BLINK_SUCCESS;
}

static blink_result_t alloc_comm_common(blink_comm_t c) {
  DeviceGuard g(c->device);
  {
    static std::mutex mu;
    static std::set<int> loaded;  // devices whose kernels are loaded
    std::lock_guard<std::mutex> lk(mu);
    if (!loaded.count(c->device)) {
      CUDA_TRY(c, preload_kernels());
      loaded.insert(c->device);
    }
  }
  CUDA_TRY(c, cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device));
  // flag words, then the LL protocol's line areas (zero = no flag yet); one
  // allocation, so the flag mapping also maps the LL area to the peers
  c->ll_bytes = c->nranks > 1 ? ll_area_bytes(c->cfg.ll_max_bytes, c->nranks,
                                               link_graph(c) || c->probe_at_connect)
                              : 0;
  CUDA_TRY(c, cudaMalloc(&c->flags, kFlagBytes + c->ll_bytes));
  CUDA_TRY(c, cudaMemset(c->flags, 0, kFlagBytes + c->ll_bytes));
  CUDA_TRY(c, cudaDeviceSynchronize());
  return BLINK_SUCCESS;
}

blink_result_t blink_init_all(blink_comm_t* comms, int ndev, const int* devs,
                              const blink_graph_t* graph, const blink_config_t* cfg_in) {
  if (!comms || !devs || ndev < 1)
    return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "comms/devs NULL or ndev < 1");
  if (ndev > kMaxRanks)
    return fail(nullptr, BLINK_ERR_UNSUPPORTED,
                "at most " + std::to_string(kMaxRanks) + " ranks per comm");
  int ndevices = 0;
  if (cudaGetDeviceCount(&ndevices) != cudaSuccess || ndevices == 0)
    return fail(nullptr, BLINK_ERR_CUDA, "no CUDA device visible");
  for (int i = 0; i < ndev; ++i)
    if (devs[i] < 0 || devs[i] >= ndevices)
      return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT,
                  "devs[" + std::to_string(i) + "] = " + std::to_string(devs[i]) + " is not a device");
  blink_config_t cfg = resolve_cfg(cfg_in);
  Graph gr;
  std::string err;
  blink_result_t r = build_graph(graph, ndev, &gr, &err);
  if (r != BLINK_SUCCESS) return fail(nullptr, r, err);
  // probe / peer access: distinct devices must reach each other
  std::vector<int> distinct;
  for (int i = 0; i < ndev; ++i)
    if (std::find(distinct.begin(), distinct.end(), devs[i]) == distinct.end())
      distinct.push_back(devs[i]);
  for (int a : distinct)
    for (int b : distinct) {
      if (a == b) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (!can)
        return fail(nullptr, BLINK_ERR_UNSUPPORTED,
                    "no peer access from device " + std::to_string(a) + " to " + std::to_string(b));
      DeviceGuard g(a);
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(nullptr, BLINK_ERR_CUDA, std::string("enable peer access: ") + cudaGetErrorString(e));
      cudaGetLastError();
    }
  // topology probe when the caller gave no graph
  Probe probe;
  if (!graph) {
    std::vector<std::string> bus(ndev);
    for (int i = 0; i < ndev; ++i) {
      char b[32] = {};
      if (cudaDeviceGetPCIBusId(b, sizeof b, devs[i]) != cudaSuccess)
        return fail(nullptr, BLINK_ERR_CUDA, "cudaDeviceGetPCIBusId failed");
      bus[i] = b;
    }
    r = probe_topology(bus, &probe, &err);
    if (r != BLINK_SUCCESS) return fail(nullptr, r, err);
    apply_probe(probe, &gr);
  }
  Clique* q = new Clique();
  q->nranks = ndev;
  q->devices = distinct;
  q->pending.resize(ndev);
  for (int i = 0; i < ndev; ++i) {
    blink_comm_t c = new blink_comm();
    c->nranks = ndev;
    c->rank = i;
    c->device = devs[i];
    c->cfg = cfg;
    c->graph = gr;
    c->probe = probe;
    c->clique = q;
    c->connected = true;
    r = alloc_comm_common(c);
    if (r != BLINK_SUCCESS) {
      g_last_error = c->last_error;
      return r;
    }
    q->comms.push_back(c);
    comms[i] = c;
  }
  // NEXT-1: one multicast object over the ranks' devices (one rank per device)
  if (cfg.nvls) {
    std::string nerr;
    std::vector<NvlsMem> mems;
    if (ndev < 2 || int(distinct.size()) != ndev) {
      nerr = "needs one rank per device on >= 2 devices";
    } else if (nvls_setup_single(std::vector<int>(devs, devs + ndev), cfg.nvls_bytes, &mems, &nerr)) {
      for (int i = 0; i < ndev; ++i) {
        q->comms[i]->nvls = mems[i];
        q->comms[i]->nvls_on = true;
        q->comms[i]->nvls_note = "on";
      }
      q->nvls = true;
    } else {
      for (auto& m : mems) nvls_release(&m);
    }
    if (!q->nvls)
      for (blink_comm* c : q->comms) c->nvls_note = "off: " + nerr;
  }
  q->per_rank = cfg.launch_per_rank != 0 && ndev > 1;
  for (int d : distinct) {
    uint64_t mask = 0;
    for (int v = 0; v < ndev; ++v)
      if (devs[v] == d) mask |= uint64_t(1) << v;
    if (!q->per_rank) {
      q->groups.push_back({d, d, mask});
      continue;
    }
    for (int v = 0; v < ndev; ++v)
      if ((mask >> v) & 1) q->groups.push_back({v, d, uint64_t(1) << v});
  }
  if (q->per_rank) {
    q->rstream.resize(ndev);
    q->rfork.resize(ndev);
    q->rjoin.resize(ndev);
    for (int v = 0; v < ndev; ++v) {
      DeviceGuard g(devs[v]);
      if (cudaStreamCreateWithFlags(&q->rstream[v], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&q->rfork[v], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&q->rjoin[v], cudaEventDisableTiming) != cudaSuccess)
        return fail(nullptr, BLINK_ERR_CUDA, "per-rank stream allocation failed");
    }
  }
  for (const Clique::Group& grp : q->groups) {
    const int d = grp.device;
    DeviceGuard g(d);
    int* h = nullptr;
    int* dp = nullptr;
    if (cudaHostAlloc(&h, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&dp, h, 0) != cudaSuccess)
      return fail(nullptr, BLINK_ERR_CUDA, "mapped error word allocation failed");
    *h = 0;
    q->err_host[grp.key] = h;
    q->err_dev[grp.key] = dp;
    uint64_t* ctrl = nullptr;
    const size_t cb = 2 * sizeof(uint64_t) + kMaxCounters * sizeof(unsigned int);
    if (cudaMalloc(&ctrl, cb) != cudaSuccess || cudaMemset(ctrl, 0, cb) != cudaSuccess)
      return fail(nullptr, BLINK_ERR_CUDA, "control word allocation failed");
    q->ctrl[grp.key] = ctrl;
  }
  q->alive = ndev;
  return BLINK_SUCCESS;
}

blink_result_t blink_init(blink_comm_t* comm, int nranks, int rank, int cuda_device,
                          const blink_graph_t* graph, const blink_config_t* cfg_in) {
  if (!comm) return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "comm is NULL");
  if (nranks < 1 || nranks > kMaxRanks)
    return fail(nullptr, BLINK_ERR_UNSUPPORTED, "nranks out of range [1,16]");
  if (rank < 0 || rank >= nranks) return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "rank out of range");
  blink_comm_t c = new blink_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = cuda_device;
  c->cfg = resolve_cfg(cfg_in);
  c->multiprocess = true;
  std::string err;
  blink_result_t r = build_graph(graph, nranks, &c->graph, &err);
  if (r != BLINK_SUCCESS) {
    delete c;
    return fail(nullptr, r, err);
  }
  c->probe_at_connect = graph == nullptr && nranks > 1;
  r = alloc_comm_common(c);
  if (r != BLINK_SUCCESS) {
    g_last_error = c->last_error;
    delete c;
    return r;
  }
  DeviceGuard g(c->device);
  CUDA_TRY(c, cudaMalloc(&c->staging, c->cfg.staging_bytes));
  c->staging_bytes = c->cfg.staging_bytes;
  if (c->cfg.nvls && nranks >= 2 && rank == 0) {  // NEXT-1: the multicast object, shared at connect
    std::string nerr;
    const size_t size = nvls_round(nranks, c->cfg.nvls_bytes);
    const int share = nvls_fabric_supported(cuda_device) ? kNvlsFabric : kNvlsPosixFd;
    if (!nvls_supported(cuda_device, share, &nerr) || !nvls_create(nranks, size, share, &c->nvls, &nerr)) {
      c->nvls_note = "off: " + nerr;
      nvls_release(&c->nvls);
    }
  }
  CUDA_TRY(c, cudaHostAlloc(&c->err_host, sizeof(int), cudaHostAllocMapped));
  CUDA_TRY(c, cudaHostGetDevicePointer(&c->err_dev, c->err_host, 0));
  *c->err_host = 0;
  const size_t cb = 2 * sizeof(uint64_t) + kMaxCounters * sizeof(unsigned int);
  CUDA_TRY(c, cudaMalloc(&c->ctrl, cb));
  CUDA_TRY(c, cudaMemset(c->ctrl, 0, cb));
  CUDA_TRY(c, cudaDeviceSynchronize());
  *comm = c;
  return BLINK_SUCCESS;
}

// NEXT-1 across processes: every rank joins rank 0's multicast object, the
// ranks meet (setup words in each other's flags: 1 = ok, 9 = failed), bind
// their memory and map it, and meet again.  NVLS turns on only when every
// rank reported ok in both rounds, so all ranks decide alike.
blink_result_t setup_barrier(blink_comm_t comm, int round, bool ok, bool* all_ok) {
  const uint64_t mine = ok ? 1 : 9;
  for (int u = 0; u < comm->nranks; ++u)
    CUDA_TRY(comm, cudaMemcpy(comm->peer_flags[u] + setup_idx(round, comm->rank), &mine, sizeof mine,
                              cudaMemcpyHostToDevice));
  std::vector<uint64_t> w(comm->nranks, 0);
  const auto t0 = std::chrono::steady_clock::now();
  while (true) {
    CUDA_TRY(comm, cudaMemcpy(w.data(), comm->flags + setup_idx(round, 0), sizeof(uint64_t) * comm->nranks,
                              cudaMemcpyDeviceToHost));
    bool all = true;
    for (uint64_t x : w) all = all && x != 0;
    if (all) break;
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > comm->cfg.timeout_s)
      return fail(comm, BLINK_ERR_TIMEOUT, "NVLS set-up: a rank did not reach barrier " + std::to_string(round));
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
  *all_ok = true;
  for (uint64_t x : w) *all_ok = *all_ok && x == 1;
  return BLINK_SUCCESS;
}

// kNvlsPosixFd: duplicate rank 0's exported fd into this process (same node,
// ptrace access to rank 0's process); -1 with *err on failure
int dup_peer_fd(int pid, int fd, std::string* err) {
  const int pidfd = int(syscall(SYS_pidfd_open, pid, 0));
  if (pidfd < 0) {
    *err = std::string("pidfd_open(rank 0): ") + strerror(errno);
    return -1;
  }
  const int lfd = int(syscall(SYS_pidfd_getfd, pidfd, fd, 0));
  if (lfd < 0)
    *err = std::string("pidfd_getfd(rank 0): ") + strerror(errno) +
           " (POSIX-fd NVLS needs ptrace access to rank 0's process)";
  close(pidfd);
  return lfd;
}

blink_result_t mp_nvls_connect(blink_comm_t comm, const Blob& b0) {
  // rank 0 keeps its own reason (set when creating / exporting the object)
  std::string nerr = comm->rank == 0 && comm->nvls_note.rfind("off: ", 0) == 0
                         ? comm->nvls_note.substr(5)
                         : "rank 0 offered no multicast object";
  bool ok = b0.nvls_offer == kNvlsFabric || b0.nvls_offer == kNvlsPosixFd;
  if (ok && comm->rank != 0) {
    ok = nvls_supported(comm->device, b0.nvls_offer, &nerr);
    if (ok && b0.nvls_offer == kNvlsPosixFd) {
      int fd = -1;
      memcpy(&fd, b0.nvls_handle, sizeof fd);
      const int lfd = dup_peer_fd(b0.pid, fd, &nerr);
      ok = lfd >= 0;
      if (ok) {
        unsigned char h[64] = {};
        memcpy(h, &lfd, sizeof lfd);
        ok = nvls_import(h, kNvlsPosixFd, size_t(b0.nvls_size), &comm->nvls, &nerr);
        close(lfd);  // the imported handle holds its own reference
      }
    } else if (ok) {
      ok = nvls_import(b0.nvls_handle, kNvlsFabric, size_t(b0.nvls_size), &comm->nvls, &nerr);
    }
  }
  if (ok) ok = nvls_add_device(&comm->nvls, comm->device, &nerr);
  bool all = false;
  blink_result_t r = setup_barrier(comm, 0, ok, &all);
  if (r != BLINK_SUCCESS) return r;
  bool ok2 = all && nvls_bind_map(&comm->nvls, comm->device, &nerr);
  if (all && !ok2) nerr = "bind/map: " + nerr;
  if (!all && ok) nerr = "another rank failed to join the multicast object";
  bool all2 = false;
  r = setup_barrier(comm, 1, ok2, &all2);
  if (r != BLINK_SUCCESS) return r;
  comm->nvls_on = all2;
  if (all2) {
    comm->nvls_note = "on";
  } else {
    if (!ok2 && all) nerr = "another rank failed to bind";
    comm->nvls_note = "off: " + nerr;
    nvls_release(&comm->nvls);
  }
  return BLINK_SUCCESS;
}

blink_result_t blink_export_handle(blink_comm_t comm, void* blob, size_t* blob_bytes) {
  if (!comm || !blob_bytes) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!comm->multiprocess) return fail(comm, BLINK_ERR_INVALID_USAGE, "not a multi-process comm");
  size_t cap = *blob_bytes;
  *blob_bytes = sizeof(Blob);
  if (!blob || cap < sizeof(Blob)) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "blob too small");
  Blob b{};
  memcpy(b.magic, "BLINKv1", 8);
  b.rank = comm->rank;
  b.nranks = comm->nranks;
  b.device = comm->device;
  b.pid = int(getpid());
  DeviceGuard g(comm->device);
  CUDA_TRY(comm, cudaDeviceGetPCIBusId(b.bus_id, sizeof b.bus_id, comm->device));
  CUDA_TRY(comm, cudaIpcGetMemHandle(&b.flags_h, comm->flags));
  CUDA_TRY(comm, cudaIpcGetMemHandle(&b.staging_h, comm->staging));
  b.staging_bytes = comm->staging_bytes;
  b.ll_bytes = comm->ll_bytes;
  b.ll_max_bytes = comm->ll_bytes ? comm->cfg.ll_max_bytes : 0;
  b.shallow_max_bytes = comm->cfg.shallow_max_bytes;
  b.onehop_bcast_max_bytes = comm->cfg.onehop_bcast_max_bytes;
  b.chunk_fp = chunking_fingerprint(comm);
  if (comm->rank == 0 && comm->nvls.mc) {
    std::string nerr;
    if (nvls_export(&comm->nvls, b.nvls_handle, &nerr)) {
      b.nvls_offer = comm->nvls.share;
      b.nvls_size = comm->nvls.size;
    } else {
      comm->nvls_note = "off: " + nerr;
    }
  }
  memcpy(blob, &b, sizeof b);
  return BLINK_SUCCESS;
}

blink_result_t blink_connect(blink_comm_t comm, const void* all_blobs, size_t blob_bytes) {
  if (!comm || !all_blobs) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!comm->multiprocess) return fail(comm, BLINK_ERR_INVALID_USAGE, "not a multi-process comm");
  if (blob_bytes < sizeof(Blob)) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "blob_bytes too small");
  DeviceGuard g(comm->device);
  const char* base = static_cast<const char*>(all_blobs);
  for (int u = 0; u < comm->nranks; ++u) {
    Blob b;
    memcpy(&b, base + size_t(u) * blob_bytes, sizeof b);
    if (memcmp(b.magic, "BLINKv1", 8) != 0 || b.rank != u || b.nranks != comm->nranks)
      return fail(comm, BLINK_ERR_INVALID_USAGE,
                  "blob " + std::to_string(u) + " is not rank " + std::to_string(u) + "'s handle");
    if (b.staging_bytes != comm->staging_bytes)
      return fail(comm, BLINK_ERR_INVALID_USAGE, "staging_bytes differs across ranks");
    if (b.ll_bytes != comm->ll_bytes ||
        b.ll_max_bytes != (comm->ll_bytes ? comm->cfg.ll_max_bytes : 0))
      return fail(comm, BLINK_ERR_INVALID_USAGE, "ll_max_bytes differs across ranks");
    if (b.shallow_max_bytes != comm->cfg.shallow_max_bytes ||
        b.onehop_bcast_max_bytes != comm->cfg.onehop_bcast_max_bytes)
      return fail(comm, BLINK_ERR_INVALID_USAGE,
                  "shallow_max_bytes / onehop_bcast_max_bytes differ across ranks");
    if (b.chunk_fp != chunking_fingerprint(comm))
      return fail(comm, BLINK_ERR_INVALID_USAGE,
                  "rank " + std::to_string(u) +
                      " chunks differently (cfg.chunk_bytes / ctas / threads / autotune, SM count or "
                      "BLINK_* chunking overrides differ)");
    if (u == comm->rank) {
      comm->peer_flags[u] = comm->flags;
      comm->peer_staging[u] = comm->staging;
      continue;
    }
    // probe: the peer GPU must be reachable (same GPU or peer access)
    int pdev = -1;
    if (cudaDeviceGetByPCIBusId(&pdev, b.bus_id) == cudaSuccess && pdev != comm->device) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, comm->device, pdev);
      if (!can)
        return fail(comm, BLINK_ERR_UNSUPPORTED,
                    "no peer access to rank " + std::to_string(u) + " (" + b.bus_id + ")");
    }
    cudaGetLastError();
    char* p = nullptr;
    blink_result_t r = open_handle(comm, b.flags_h, &p);
    if (r != BLINK_SUCCESS) return r;
    comm->peer_flags[u] = reinterpret_cast<uint64_t*>(p);
    r = open_handle(comm, b.staging_h, &p);
    if (r != BLINK_SUCCESS) return r;
    comm->peer_staging[u] = p;
  }
  if (comm->cfg.nvls && comm->nranks >= 2) {  // NEXT-1 set-up: join, barrier, bind, barrier
    Blob b0;
    memcpy(&b0, base, sizeof b0);
    blink_result_t nr = mp_nvls_connect(comm, b0);
    if (nr != BLINK_SUCCESS) return nr;
  }
  if (comm->probe_at_connect) {  // topology probe over every rank's GPU
    std::vector<std::string> bus(comm->nranks);
    for (int u = 0; u < comm->nranks; ++u) {
      Blob b;
      memcpy(&b, base + size_t(u) * blob_bytes, sizeof b);
      bus[u] = b.bus_id;
    }
    std::string perr;
    blink_result_t pr = probe_topology(bus, &comm->probe, &perr);
    if (pr != BLINK_SUCCESS) return fail(comm, pr, perr);
    apply_probe(comm->probe, &comm->graph);
    comm->plans.clear();
  }
  Reg st;
  st.buf = comm->staging;
  st.bytes = comm->staging_bytes;
  for (int u = 0; u < comm->nranks; ++u) st.peer[u] = comm->peer_staging[u];
  comm->regs.push_back(st);
  comm->connected = true;
  return BLINK_SUCCESS;
}

blink_result_t blink_register_export(blink_comm_t comm, void* buf, size_t bytes, void* blob,
                                     size_t* blob_bytes) {
  if (!comm || !blob_bytes) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL argument");
  size_t cap = *blob_bytes;
  *blob_bytes = sizeof(RegBlob);
  if (!comm->multiprocess || !blob) return BLINK_SUCCESS;  // blob == NULL: size query
  if (cap < sizeof(RegBlob)) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "blob too small");
  if (!buf || bytes == 0) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "empty buffer");
  DeviceGuard g(comm->device);
  // allocation base of `buf` (IPC handles name whole allocations); the driver
  // symbol is fetched through the runtime so the library never links libcuda.
  typedef CUresult (*GetRange)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    CUDA_TRY(comm, cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &qr));
    if (!fn) return fail(comm, BLINK_ERR_CUDA, "cuMemGetAddressRange entry point not found");
    get_range = reinterpret_cast<GetRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult cr = get_range(&base, &size, reinterpret_cast<CUdeviceptr>(buf));
  if (cr != CUDA_SUCCESS) return fail(comm, BLINK_ERR_CUDA, "cuMemGetAddressRange failed");
  RegBlob rb{};
  memcpy(rb.magic, "BLINKrg", 8);
  rb.rank = comm->rank;
  rb.bytes = bytes;
  if (cudaIpcGetMemHandle(&rb.h, reinterpret_cast<void*>(base)) == cudaSuccess) {
    rb.kind = 0;
    rb.offset = uint64_t(reinterpret_cast<char*>(buf) - reinterpret_cast<char*>(base));
  } else {  // VMM memory (e.g. PyTorch expandable segments): export every chunk
    cudaGetLastError();
    std::vector<VmmChunk> ch;
    std::string verr;
    if (!vmm_chunks(buf, bytes, &ch, &verr))
      return fail(comm, BLINK_ERR_UNSUPPORTED,
                  "buffer is neither cudaMalloc memory nor an exportable VMM allocation: " + verr);
    if (int(ch.size()) > kMaxVmmChunks) {
      for (auto& c : ch) close(c.fd);
      return fail(comm, BLINK_ERR_UNSUPPORTED, "buffer spans more than 128 VMM chunks");
    }
    rb.kind = 1;
    rb.pid = int32_t(getpid());
    rb.nchunks = int32_t(ch.size());
    for (size_t i = 0; i < ch.size(); ++i) {
      rb.chunks[i].off = ch[i].off;
      rb.chunks[i].size = ch[i].size;
      rb.chunks[i].fd = ch[i].fd;
      comm->exported_fds.push_back(ch[i].fd);
    }
  }
  memcpy(blob, &rb, sizeof rb);
  return BLINK_SUCCESS;
}

blink_result_t blink_register_connect(blink_comm_t comm, void* buf, const void* all_blobs,
                                      size_t blob_bytes) {
  if (!comm) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL comm");
  if (!comm->multiprocess) return BLINK_SUCCESS;
  if (!all_blobs || blob_bytes < sizeof(RegBlob))
    return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "bad blobs");
  DeviceGuard g(comm->device);
  Reg reg;
  reg.buf = static_cast<char*>(buf);
  const char* base = static_cast<const char*>(all_blobs);
  for (int u = 0; u < comm->nranks; ++u) {
    RegBlob rb;
    memcpy(&rb, base + size_t(u) * blob_bytes, sizeof rb);
    if (memcmp(rb.magic, "BLINKrg", 8) != 0 || rb.rank != u)
      return fail(comm, BLINK_ERR_INVALID_USAGE, "registration blob " + std::to_string(u) + " is invalid");
    if (u == 0) reg.bytes = rb.bytes;
    if (rb.bytes != reg.bytes)
      return fail(comm, BLINK_ERR_INVALID_USAGE, "registered sizes differ across ranks (symmetric registration)");
    if (u == comm->rank) {
      reg.peer[u] = reg.buf;
      continue;
    }
    if (rb.kind == 1) {  // VMM chunks: duplicate the exporter's fds, map them back to back
      if (rb.nchunks <= 0 || rb.nchunks > kMaxVmmChunks)
        return fail(comm, BLINK_ERR_INVALID_USAGE, "registration blob " + std::to_string(u) + " is invalid");
      const int pidfd = int(syscall(SYS_pidfd_open, rb.pid, 0));
      if (pidfd < 0)
        return fail(comm, BLINK_ERR_SYSTEM, "pidfd_open(rank " + std::to_string(u) + "): " + strerror(errno));
      std::vector<VmmChunk> ch(rb.nchunks);
      std::vector<int> lfds;
      for (int i = 0; i < rb.nchunks; ++i) {
        ch[i].off = rb.chunks[i].off;
        ch[i].size = rb.chunks[i].size;
        ch[i].fd = rb.chunks[i].fd;
        const int lfd = int(syscall(SYS_pidfd_getfd, pidfd, rb.chunks[i].fd, 0));
        if (lfd < 0) {
          const std::string why = strerror(errno);
          for (int f : lfds) close(f);
          close(pidfd);
          return fail(comm, BLINK_ERR_SYSTEM,
                      "pidfd_getfd(rank " + std::to_string(u) + "): " + why +
                          " (VMM registration needs ptrace access to the peer process)");
        }
        lfds.push_back(lfd);
      }
      close(pidfd);
      VmmMapping m;
      std::string verr;
      const bool ok = vmm_map_peer(ch, lfds, comm->device, &m, &verr);
      for (int f : lfds) close(f);
      if (!ok) {
        vmm_unmap(&m);
        return fail(comm, BLINK_ERR_CUDA, "mapping rank " + std::to_string(u) + "'s VMM chunks: " + verr);
      }
      reg.peer[u] = m.base;
      comm->vmm_maps.push_back(m);
      continue;
    }
    char* p = nullptr;
    blink_result_t r = open_handle(comm, rb.h, &p);
    if (r != BLINK_SUCCESS) return r;
    reg.peer[u] = p + rb.offset;
  }
  comm->regs.push_back(reg);
  return BLINK_SUCCESS;
}

blink_result_t blink_broadcast(blink_comm_t comm, const void* sendbuf, void* recvbuf, size_t count,
                               blink_dtype_t dtype, int root, void* stream) {
  blink_result_t r = validate_call(comm, count, dtype, BLINK_SUM, root, kBroadcast);
  if (r != BLINK_SUCCESS) return r;
  if (count > 0 && (!recvbuf || (comm->rank == root && !sendbuf)))
    return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (comm->multiprocess) {
    if (count == 0) return BLINK_SUCCESS;
    return mp_collective(comm, kBroadcast, sendbuf, recvbuf, count, dtype, BLINK_SUM, root, stream);
  }
  return clique_post(comm, kBroadcast, sendbuf, recvbuf, count, dtype, BLINK_SUM, root, stream);
}

blink_result_t blink_allreduce(blink_comm_t comm, const void* sendbuf, void* recvbuf, size_t count,
                               blink_dtype_t dtype, blink_redop_t op, void* stream) {
  blink_result_t r = validate_call(comm, count, dtype, op, 0, kAllReduce);
  if (r != BLINK_SUCCESS) return r;
  if (count > 0 && (!recvbuf || !sendbuf))
    return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (comm->multiprocess) {
    if (count == 0) return BLINK_SUCCESS;
    return mp_collective(comm, kAllReduce, sendbuf, recvbuf, count, dtype, op, -1, stream);
  }
  return clique_post(comm, kAllReduce, sendbuf, recvbuf, count, dtype, op, -1, stream);
}

blink_result_t blink_reduce_scatter(blink_comm_t comm, const void* sendbuf, void* recvbuf,
                                    size_t recvcount, blink_dtype_t dtype, blink_redop_t op,
                                    void* stream) {
  blink_result_t r = validate_call(comm, recvcount, dtype, op, 0, kReduceScatter);
  if (r != BLINK_SUCCESS) return r;
  if (recvcount > 0 && (!recvbuf || !sendbuf))
    return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (comm->multiprocess) {
    if (recvcount == 0) return BLINK_SUCCESS;
    return mp_collective(comm, kReduceScatter, sendbuf, recvbuf, recvcount, dtype, op, -1, stream);
  }
  return clique_post(comm, kReduceScatter, sendbuf, recvbuf, recvcount, dtype, op, -1, stream);
}

blink_result_t blink_allgather(blink_comm_t comm, const void* sendbuf, void* recvbuf,
                               size_t sendcount, blink_dtype_t dtype, void* stream) {
  blink_result_t r = validate_call(comm, sendcount, dtype, BLINK_SUM, 0, kAllGather);
  if (r != BLINK_SUCCESS) return r;
  if (sendcount > 0 && (!recvbuf || !sendbuf))
    return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (comm->multiprocess) {
    if (sendcount == 0) return BLINK_SUCCESS;
    return mp_collective(comm, kAllGather, sendbuf, recvbuf, sendcount, dtype, BLINK_SUM, -1, stream);
  }
  return clique_post(comm, kAllGather, sendbuf, recvbuf, sendcount, dtype, BLINK_SUM, -1, stream);
}

blink_result_t blink_gather(blink_comm_t comm, const void* sendbuf, void* recvbuf,
                            size_t sendcount, blink_dtype_t dtype, int root, void* stream) {
  blink_result_t r = validate_call(comm, sendcount, dtype, BLINK_SUM, root, kGather);
  if (r != BLINK_SUCCESS) return r;
  if (sendcount > 0 && (!sendbuf || (comm->rank == root && !recvbuf)))
    return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (comm->multiprocess) {
    if (sendcount == 0) return BLINK_SUCCESS;
    return mp_collective(comm, kGather, sendbuf, recvbuf, sendcount, dtype, BLINK_SUM, root, stream);
  }
  return clique_post(comm, kGather, sendbuf, recvbuf, sendcount, dtype, BLINK_SUM, root, stream);
}

blink_result_t blink_get_plan(blink_comm_t comm, int is_allreduce, int root, size_t count,
                              blink_dtype_t dtype, char* json, size_t* json_bytes) {
  if (!comm || !json_bytes) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL argument");
  int coll = is_allreduce ? kAllReduce : kBroadcast;
  blink_result_t r = validate_call(comm, count, dtype, BLINK_SUM, root, coll);
  if (r != BLINK_SUCCESS) return r;
  const int es = esize_of(dtype);
  const Plan* plan = nullptr;
  r = get_plan(comm, coll, root, count * es, &plan);
  if (r != BLINK_SUCCESS) return r;
  // the launch this rank belongs to, and every launch group of the call
  uint64_t mask = 0;
  std::vector<uint64_t> gm;
  int share = 1;
  if (comm->multiprocess) {
    mask = uint64_t(1) << comm->rank;
    for (int u = 0; u < comm->nranks; ++u) gm.push_back(uint64_t(1) << u);
  } else {
    share = 0;
    for (const Clique::Group& g : comm->clique->groups) {
      gm.push_back(g.mask);
      if ((g.mask >> comm->rank) & 1) mask = g.mask;
      if (g.device == comm->device) ++share;
    }
  }
  Sized s;
  int budget = std::max(1, co_resident_budget(comm, comm->device, dtype, BLINK_SUM, coll) / share);
  r = build_sized(comm, *plan, count, es, mask, gm, budget, &s);
  if (r != BLINK_SUCCESS) return r;
  std::string j = plan_to_json(*plan, count, es, s.ranges, s.ctas);
  j.insert(j.size() - 1, ",\"topology\":" + probe_to_json(comm->probe));
  {
    const bool would = comm->nvls_on && nvls_call(coll, BLINK_SUM) &&
                       !ll_tree(comm, *plan, coll, count * es);
    std::string note = comm->nvls_note;
    for (char& ch : note)
      if (ch == '"') ch = '\'';
    j.insert(j.size() - 1, std::string(",\"nvls\":{\"active\":") + (comm->nvls_on ? "true" : "false") +
                               ",\"this_call\":" + (would ? "true" : "false") + ",\"note\":\"" + note + "\"}");
  }
  size_t need = j.size() + 1, cap = *json_bytes;
  *json_bytes = need;
  if (!json || cap < need) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "json buffer too small");
  memcpy(json, j.c_str(), need);
  return BLINK_SUCCESS;
}

blink_result_t blink_get_trace(blink_comm_t comm, uint64_t* out, size_t* n_words) {
  if (!comm || !n_words) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL argument");
  const int key = comm->multiprocess ? -1 : (comm->clique->per_rank ? comm->rank : comm->device);
  if (comm->multiprocess || !comm->clique->trace.count(key)) {
    *n_words = 0;
    return BLINK_SUCCESS;
  }
  const size_t need = size_t(comm->clique->trace_ctas[key]) * kTraceSlots;
  const size_t cap = *n_words;
  *n_words = need;
  if (!out || cap < need) return BLINK_SUCCESS;
  DeviceGuard g(comm->device);
  CUDA_TRY(comm, cudaMemcpy(out, comm->clique->trace[key], need * sizeof(uint64_t),
                            cudaMemcpyDeviceToHost));
  return BLINK_SUCCESS;
}

blink_result_t blink_get_stats(blink_comm_t comm, blink_stats_t* st) {
  if (!comm || !st) return fail(comm, BLINK_ERR_INVALID_ARGUMENT, "NULL argument");
  *st = comm->stats;
  return BLINK_SUCCESS;
}

blink_result_t blink_comm_info(blink_comm_t comm, int* nranks, int* rank, int* device) {
  if (!comm) return fail(nullptr, BLINK_ERR_INVALID_ARGUMENT, "NULL comm");
  if (nranks) *nranks = comm->nranks;
  if (rank) *rank = comm->rank;
  if (device) *device = comm->device;
  return BLINK_SUCCESS;
}

blink_result_t blink_destroy(blink_comm_t comm) {
  if (!comm) return BLINK_SUCCESS;
  {
    DeviceGuard g(comm->device);
    cudaDeviceSynchronize();
    if (comm->multiprocess) {
      for (auto& kv : comm->sized) {
        cudaFree(kv.second.d_tasks);
        cudaFree(kv.second.d_trees);
      }
      for (auto& kv : comm->opened) cudaIpcCloseMemHandle(kv.second);
      for (auto& m : comm->vmm_maps) vmm_unmap(&m);
      for (int f : comm->exported_fds) close(f);
      if (comm->staging) cudaFree(comm->staging);
      for (auto& kv : comm->mp_miad) {
        if (kv.second.ev0) cudaEventDestroy(kv.second.ev0);
        if (kv.second.ev1) cudaEventDestroy(kv.second.ev1);
      }
      if (comm->miad_stream) cudaStreamDestroy(comm->miad_stream);
      if (comm->err_host) cudaFreeHost(comm->err_host);
      if (comm->ctrl) cudaFree(comm->ctrl);
    }
    if (comm->flags) cudaFree(comm->flags);
    if (comm->scratch) cudaFree(comm->scratch);
    if (comm->nvls.mc) nvls_release(&comm->nvls);
  }
  Clique* q = comm->clique;
  if (q) {
    bool last = false;
    {
      std::lock_guard<std::mutex> lk(q->mu);
      last = --q->alive == 0;
    }
    if (last) {
      for (auto& kv : q->sized) {
        cudaFree(kv.second.d_tasks);
        cudaFree(kv.second.d_trees);
      }
      for (auto& kv : q->err_host) cudaFreeHost(kv.second);
      for (auto& kv : q->ctrl) cudaFree(kv.second);
      for (auto& kv : q->trace) cudaFree(kv.second);
      for (auto st : q->rstream) cudaStreamDestroy(st);
      for (auto ev : q->rfork) cudaEventDestroy(ev);
      for (auto ev : q->rjoin) cudaEventDestroy(ev);
      for (auto& kv : q->miad) {
        if (kv.second.ev0) cudaEventDestroy(kv.second.ev0);
        if (kv.second.ev1) cudaEventDestroy(kv.second.ev1);
      }
      delete q;
    }
  }
  delete comm;
  return BLINK_SUCCESS;
}

}  // extern "C"
