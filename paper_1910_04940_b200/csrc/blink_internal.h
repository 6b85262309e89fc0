// Internal structures shared by the control plane (plan.cpp), the host
// runtime (runtime.cpp) and the device executor (exec.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/blink.h"

namespace blink {

// ---------------------------------------------------------------- limits
constexpr int kMaxRanks = 16;       // ranks per comm (one NVSwitch node; DGX-2 = 16)
constexpr int kMaxTrees = 32;       // trees per plan
constexpr int kMaxChunks = 512;     // chunks per tree per call
constexpr int kGrain = 16;
constexpr int kTraceSlots = 16;     // per-CTA trace stamps (BLINK_TRACE)
constexpr int kMaxCounters = 4096;  // dynamic chunk counters per launch (ctrl[2..])          // split grain in bytes (R#11) == one 128-bit vector

// Flag region of one rank (uint64 words, monotonically increasing epochs,
// never reset).  Producers write into the CONSUMER's region:
//   entry[u]              rank u entered call `epoch` (its send is ready and
//                         its recv may be overwritten)
//   pflag[i][u][c]        child u's partial for tree i / chunk c is ready
//                         (written by u into its parent's region)
//   bflag[i][c]           the final value of tree i / chunk c has been
//                         written into this rank's recv (written by parent)
//   miad[s]               (multi-process MIAD, NEXT-2) rank 0's chunk decision for
//                         autotuned call s: {s + 1, chunk | phase << 56}, slot s % kMiadSlots
constexpr size_t kEntryWords = kMaxRanks;
constexpr size_t kPflagWords = size_t(kMaxTrees) * kMaxRanks * kMaxChunks;
constexpr size_t kBflagWords = size_t(kMaxTrees) * kMaxChunks;
constexpr size_t kMiadSlots = 64;
constexpr size_t kMiadWords = 2 * kMiadSlots;
//   setup[2][u]           NVLS set-up barriers at blink_connect (1 = ok, 9 = failed)
constexpr size_t kSetupWords = 2 * kMaxRanks;
constexpr size_t kFlagWords = kEntryWords + kPflagWords + kBflagWords + kMiadWords + kSetupWords;
constexpr size_t kFlagBytes = kFlagWords * sizeof(uint64_t);
__host__ __device__ inline size_t entry_idx(int u) { return size_t(u); }
__host__ __device__ inline size_t pflag_idx(int tree, int child, int chunk) {
  return kEntryWords + (size_t(tree) * kMaxRanks + child) * kMaxChunks + chunk;
}
__host__ __device__ inline size_t bflag_idx(int tree, int chunk) {
  return kEntryWords + kPflagWords + size_t(tree) * kMaxChunks + chunk;
}
__host__ __device__ inline size_t miad_idx(uint64_t seq) {
  return kEntryWords + kPflagWords + kBflagWords + 2 * size_t(seq % kMiadSlots);
}
__host__ __device__ inline size_t setup_idx(int round, int u) {
  return kEntryWords + kPflagWords + kBflagWords + kMiadWords + size_t(round) * kMaxRanks + u;
}

enum Coll : int { kBroadcast = 0, kAllReduce = 1, kReduceScatter = 2, kAllGather = 3, kGather = 4 };
// ReduceScatter / AllGather / Gather: tree j is the one-hop star rooted at j and owns block j
// (Gather: the star has the single leaf `root`; other ranks are not members, parent -2).
inline bool is_block_coll(int c) { return c == kReduceScatter || c == kAllGather || c == kGather; }
// collectives whose tree roots push their own send down the tree
inline __host__ __device__ bool is_push_coll(int c) { return c == kBroadcast || c == kAllGather || c == kGather; }

// ---------------------------------------------------------------- plans
struct Tree {
  int root = 0;
  std::vector<int> parent;   // parent[root] = -1; -2 = not in this tree (Gather)
  int64_t wnum = 1;          // weight = wnum / wden (exact rational, P:390 grid)
  int64_t wden = 1;
  int depth = 0;
};

struct Plan {                // size-independent (TreeGen output)
  int coll = kAllReduce;
  int root = -1;             // broadcast root, -1 for AllReduce
  int nranks = 0;
  std::vector<Tree> trees;   // in split order (R#11)
  int64_t rate_num = 0, rate_den = 1;
  double c_star = 0.0;       // best MWU rate (0 for closed forms)
  double opt = 0.0;          // optimal rate the ILP ladder is measured against (R#3)
  bool accepted = true;      // the ladder reached (1 - gap) * opt
  int grid = 1;              // accepted relaxation level g
  bool switch_model = false;
  bool blocks = false;       // tree i covers block i = [i*count, (i+1)*count) (RS / AG)
};

struct TreeRange {           // per call size
  int64_t lo = 0, hi = 0;    // element range [lo, hi)
  int64_t chunk = 0;         // elements per chunk
  int nchunks = 0;
};

// Role of one CTA (a "channel" slice, a6).
enum Role : int {
  kRoleReduce = 0,  // AllReduce: combine own send + children, forward to parent
                    // (or, at the root, write the result and push it down)
  kRoleBcast = 1,   // forward a chunk down the tree (Broadcast, AllReduce phase 2)
  kRoleExit = 2,    // only entry/exit bookkeeping for this rank
};

struct DevTree {             // 40 bytes; byte offsets into every rank's buffers
  int64_t lo, hi, chunk;
  int32_t nchunks;
  int32_t root;
  uint32_t members;          // ranks in the tree (Gather trees span root + one leaf)
  int32_t pad;
};

struct DevTask {             // one per CTA segment; 104 bytes
  int16_t rank;              // acting rank v
  int16_t tree;              // tree index i
  int16_t role;
  int16_t parent;            // -1 at the tree root
  uint32_t children;         // bitmask of v's children in tree i
  uint32_t leafmask;         // children that are leaves (their send is read directly)
  int32_t cta_idx, cta_cnt;  // position among the CTAs of this (rank, tree, role)
  int32_t exit_idx, exit_cnt;// position among the CTAs of rank v (exit wait split)
  int32_t do_entry;          // this task publishes rank v's entry flag
  int32_t next;              // next task (segment) of the same CTA, -1 = none
  int32_t c0, c1, cstride;   // chunks c = c0, c0+cstride, ... < c1 of tree `tree`
  int32_t ctr;               // >= 0: chunks are taken from counter ctrl[2 + ctr] (dynamic)
  int32_t merged;            // chunk ids span every tree (one-hop AllReduce, single launch)
  int32_t pad1;
  DevTree tr;                // copy of trees[tree] (saves a dependent load at launch)
};
static_assert(sizeof(DevTask) == 104, "DevTask layout");



constexpr int kMaxArgRanks = kMaxRanks;
struct LaunchArgs {
  const DevTask* tasks;
  const DevTree* trees;
  int ntrees;
  int nranks;
  int coll;                  // Coll
  int dtype;                 // blink_dtype_t
  int op;                    // blink_redop_t
  int exit_wait;             // 1 when ranks live in different launches
  int bcast_root;            // Broadcast root rank
  int use_tma;               // stage aligned bodies through TMA bulk copies
  int smem_bytes;            // dynamic shared memory of the TMA ring
  int tile_bytes;            // 0 = default tile per source
  int scope_sys;             // 1: flags cross devices/processes (.sys), 0: one device (.gpu)
  int store_depth;           // bulk-store groups kept in flight (-1 = default)
  int l2_hint;               // 1: TMA loads/stores carry an L2 evict-first policy
  int defer_signal;          // 1: chunk signals wait for their own bulk group only (no drain)
  uint64_t* trace;           // BLINK_TRACE: kTraceSlots globaltimer stamps per CTA, else NULL
  int nctr;                  // chunk counters ctrl[2 .. 2 + nctr) zeroed by the last CTA
  int split_ring;            // 1: signalling copies alternate chunks over two store threads
  int copy_stages;           // stage-ring depth of copies (0 = default 6; BLINK_COPY_STAGES)
  int chan0, nchan;          // work stealing (a6): tasks[chan0 + ci] describes dynamic channel ci
                             // of this launch (cta_idx = -1: a joining CTA); nchan = 0: off
  uint64_t epoch;            // set by the kernel from ctrl[0] + 1
  uint64_t* ctrl;            // device words: [0] epoch of the last completed launch,
                             // [1] CTAs finished in the current launch (graph-safe epochs)
  uint64_t timeout_ns;
  int* err;                  // host-mapped error word (0 = ok)
  // What a CTA reads before its first TMA load sits together here (the
  // parameter bank's misses serialise, so the fields share few lines).
  int32_t merged_all;            // every CTA runs mtask (cta_idx = c0 = blockIdx.x): no task load
  int32_t pad5;
  int64_t mchunk;                // merged: chunk c = bytes [c*mchunk, min(mbytes, (c+1)*mchunk))
  int64_t mbytes;                // merged: bytes per rank
  DevTask mtask;
  char* send[kMaxArgRanks];
  char* recv[kMaxArgRanks];
  // link-graph ReduceScatter: inner ranks keep their partials of other blocks
  // in relay[v] (an m-block area, unshifted); roots write recv (NULL = unused)
  char* relay[kMaxArgRanks];
  uint64_t* flags[kMaxArgRanks];
  // Per-call tables in the parameter space (constant bank): no dependent
  // global loads before a CTA's first TMA load.
  DevTree ptrees[kMaxTrees];     // = trees[0 .. ntrees)
  int32_t tree_end[kMaxTrees];   // prefix sums of ptrees[i].nchunks
};
static_assert(sizeof(LaunchArgs) <= 4096, "kernel parameter space");

// Low-latency (LL) protocol for small calls on switch plans (NEXT-2's
// small-message protocol).  The same one-hop trees, but
// readiness travels inside the data: every 16-byte line is {d0, flag, d1,
// flag} written with one 128-bit store (each {data, flag} 8-byte half is
// single-copy atomic), the flag being the call's epoch.  A leaf pushes its
// slice j into root j's LL area, root j polls its own memory, reduces in
// ascending-rank order and pushes the result lines into every leaf's LL area;
// a leaf polls and copies out.  No rank touches a peer's user buffers, so
// there is no entry handshake and no exit wait; areas alternate by epoch
// parity (a rank cannot reach call e+2 before every peer finished reading call
// e).  Per rank, after the flag words:
//   IN [p][src][cap]   lines from leaf src for this rank's slice (parity p)
//   OUT[p][j][cap]     result lines of root j's slice (Broadcast: one
//                      contiguous run of the whole buffer from OUT[p][0])
constexpr int kLLThreads = 256;
// Link graphs (R#27) also run small calls on one tree in the LL protocol
// (LLArgs::tree): a child's whole buffer goes into one IN slot, so their slots
// hold ll_tree_max(ll_max) bytes (<= 128 KiB: A/B on DGX-1V, the tree
// executor wins beyond it for AllReduce).
inline size_t ll_tree_max(size_t ll_max_bytes) {
  const size_t t = ll_max_bytes / 2;
  return (t < (size_t(128) << 10) ? t : (size_t(128) << 10)) / 16 * 16;
}
inline size_t ll_cap_lines(size_t ll_max_bytes, int m, bool link_graph = false) {
  size_t cap = ll_max_bytes / (8 * size_t(m)) + 8;
  if (link_graph && ll_tree_max(ll_max_bytes) / 8 + 8 > cap) cap = ll_tree_max(ll_max_bytes) / 8 + 8;
  return cap;
}
inline size_t ll_area_bytes(size_t ll_max_bytes, int m, bool link_graph = false) {
  return ll_max_bytes ? 4 * size_t(m) * ll_cap_lines(ll_max_bytes, m, link_graph) * 16 : 0;
}
struct LLArgs {
  int nranks, coll, dtype, op;
  int root;                    // Broadcast root
  int nlocal;                  // ranks run by this launch: ranks[0 .. nlocal)
  int ctas_per_rank;
  int scope_sys;               // 1: peers on other devices / processes (.sys flags)
  int tree;                    // 1: one multi-level tree (R#27 shallow plan), parent[] below
  int tree_root;               // its root (AllReduce: the graph centre)
  int8_t parent[kMaxRanks];    // tree: parent rank, -1 at the root
  int8_t ranks[kMaxRanks];
  int64_t bytes;               // S per rank
  int64_t cap;                 // lines per slice area (ll_cap_lines)
  int64_t lo[kMaxRanks + 1];   // AllReduce: slice j = bytes [lo[j], lo[j+1]) (tree rooted at j)
  uint64_t* ctrl;              // launch epoch words (shared with the tree executor)
  int* err;
  uint64_t timeout_ns;
  uint64_t* trace;
  const char* send[kMaxRanks];
  char* recv[kMaxRanks];
  uint4* ll[kMaxRanks];        // rank u's LL area (peer-mapped)
};

// NEXT-1 (nvls.cu): one call / piece of an NVLS AllReduce (SUM) or Broadcast
// over the multicast-bound buffers uc (unicast) / mc (multicast) of `bytes`
// (a multiple of 16), for rank `rank`.
struct NvlsArgs {
  int nranks, rank, coll, dtype, root;
  int pad;
  int64_t bytes;
  const char* send;
  char* recv;
  char* uc;
  char* mc;
  uint64_t* flags[kMaxRanks];  // every rank's flag words (peer mappings)
  uint64_t* ctrl;              // this launch's epoch / counter words
  int* err;
  uint64_t timeout_ns;
};
cudaError_t launch_nvls(const NvlsArgs& a, int grid, void* stream);

// nvls_host.cpp: multicast objects (driver handles as 64-bit integers)
// How a multicast object crosses processes: not at all (single process), a
// FABRIC handle (IMEX / fabric manager), or a POSIX file descriptor the
// peers duplicate with pidfd_getfd (single node without FABRIC support).
enum NvlsShare { kNvlsLocal = 0, kNvlsFabric = 1, kNvlsPosixFd = 2 };
struct NvlsMem {
  unsigned long long mc = 0, mem = 0;      // multicast object, bound physical memory
  unsigned long long uc_va = 0, mc_va = 0; // unicast / multicast mappings
  size_t size = 0;
  int dev = -1;
  bool owner = false, bound = false;
  int share = kNvlsLocal;
  int export_fd = -1;  // kNvlsPosixFd exporter: kept open until release (peers duplicate it)
};
// multicast support on `dev`; `share` kNvlsFabric also needs FABRIC handles
bool nvls_supported(int dev, int share, std::string* err);
bool nvls_fabric_supported(int dev);
size_t nvls_round(int ndev, size_t bytes);
bool nvls_create(int ndev, size_t bytes, int share, NvlsMem* m, std::string* err);
// 64 bytes: the FABRIC handle, or (kNvlsPosixFd) the exporter's fd as an int
bool nvls_export(NvlsMem* m, void* handle, std::string* err);
// kNvlsPosixFd: `handle` holds a fd valid in THIS process (duplicated by the caller)
bool nvls_import(const void* handle, int share, size_t bytes, NvlsMem* m, std::string* err);
bool nvls_add_device(NvlsMem* m, int dev, std::string* err);
bool nvls_bind_map(NvlsMem* m, int dev, std::string* err);
void nvls_release(NvlsMem* m);
bool nvls_setup_single(const std::vector<int>& devs, size_t bytes, std::vector<NvlsMem>* out, std::string* err);
// VMM (PyTorch expandable segments) registration: the physical chunks a
// buffer touches, exported as POSIX fds, mapped back to back at a peer.
struct VmmChunk {
  int64_t off = 0;    // chunk start relative to the buffer (<= 0 for the first)
  size_t size = 0;
  int fd = -1;        // exporter's fd
};
struct VmmMapping {
  unsigned long long va = 0;
  size_t span = 0;
  char* base = nullptr;  // where the peer's buffer starts in this process
  std::vector<std::pair<unsigned long long, size_t>> mapped;
};
bool vmm_chunks(const void* buf, size_t bytes, std::vector<VmmChunk>* out, std::string* err);
bool vmm_map_peer(const std::vector<VmmChunk>& chunks, const std::vector<int>& local_fds, int dev,
                  VmmMapping* out, std::string* err);
void vmm_unmap(VmmMapping* m);

// exec.cu
cudaError_t launch_ll(const LLArgs& a, int grid, void* stream, bool cooperative, bool pdl);
cudaError_t launch_exec(const LaunchArgs& a, int grid, int threads, bool vec, void* stream,
                        bool cooperative, bool pdl);
constexpr int kMaxSmemBytes = 224 * 1024;  // + static smem <= 227 KB opt-in
cudaError_t launch_copy(void* dst, const void* src, size_t bytes, void* stream);
// force-load every kernel module on the current device (lazy loading would
// otherwise load at a first launch that may wait for spinning kernels)
cudaError_t preload_kernels();
cudaError_t preload_nvls_kernels();
// two u64 stores by one thread, stream-ordered (values travel as kernel parameters)
cudaError_t launch_store2(uint64_t* dst, uint64_t v0, uint64_t v1, void* stream);
int exec_max_ctas_per_sm(int threads, bool vec, int dtype, int op, int coll, int smem_bytes);

// plan.cpp -------------------------------------------------------------
struct Graph {
  int n = 0;                       // GPU nodes (ranks)
  bool switch_model = true;        // all GPUs behind a switch (or NULL graph)
  std::vector<std::vector<double>> cap;  // cap[u][v], directed, GPU nodes only
  // NEXT-4 multi-server: GPU-GPU links inside servers + a network SWITCH
  bool multi_server = false;
  std::vector<std::vector<int>> servers;  // rank lists, ascending
};

// Parse/validate a user graph for nranks ranks.  Returns BLINK_SUCCESS or an
// error with `err` describing the offending link/node.
blink_result_t build_graph(const blink_graph_t* g, int nranks, Graph* out, std::string* err);
blink_result_t make_plan(const Graph& g, int coll, int root, const blink_config_t& cfg, Plan* out,
                         std::string* err);
// R#27 latency plan: one minimum-depth (BFS) tree for small calls on link graphs.
bool use_shallow_plan(const Graph& g, int coll, size_t bytes, const blink_config_t& cfg);
blink_result_t make_shallow_plan(const Graph& g, int coll, int root, Plan* out, std::string* err);
// NEXT-3 on link graphs: AllGather / Gather block plans (tree j covers block j).
blink_result_t make_block_plan(const Graph& g, int coll, int root, Plan* out, std::string* err);
// Split (R#11) + chunking (a8).  ctas_for_tree: CTA count expected per tree channel.
blink_result_t size_plan(const Plan& p, size_t count, int esize, const blink_config_t& cfg,
                         int ctas_hint, std::vector<TreeRange>* out, std::string* err);
std::string plan_to_json(const Plan& p, size_t count, int esize, const std::vector<TreeRange>& r,
                         int ctas);
int esize_of(blink_dtype_t d);

// probe.cpp -------------------------------------------------------------
// Topology probe: NVLink ports of the ranks' GPUs from NVML.
struct Probe {
  std::string kind = "virtual";            // virtual | nvswitch | nvlink | pcie
  std::string note;
  std::vector<std::vector<int>> links;     // links[u][v]: NVLink ports of u ending at v
  std::vector<int> switch_ports;           // NVLink ports of u ending at an NVSwitch
};
blink_result_t probe_topology(const std::vector<std::string>& bus_ids, Probe* out, std::string* err);
void apply_probe(const Probe& p, Graph* g);  // "nvlink" -> the link graph (if connected)
std::string probe_to_json(const Probe& p);

}  // namespace blink
