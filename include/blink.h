/*
 * blink.h -- C ABI of the B200-native Blink collectives library.
 *
 * Blink (Wang et al., arXiv:1910.04940) packs spanning trees over the link
 * graph of the GPUs a job was allocated and runs Broadcast and AllReduce as
 * chunked, pipelined transfers along those trees.  Citations "P:<line>" refer
 * to PAPER.md (the paper's LaTeX) and name the section / equation.
 *
 *   - Problem statement: a graph G(V, E, c_e) of GPUs and links with
 *     bandwidth-proportional capacities, a root r (Sec. 3.1,
 *     Eqs. 1-3); the topology is probed over the allocated GPUs only.
 *   - Broadcast: the buffer is split across the packed trees in proportion to
 *     their weights, each piece is chunked and forwarded down its tree
 *     (Sec. 4.1).
 *   - AllReduce: per tree, reduce toward a chosen root, then broadcast the
 *     result back down the same tree with the links reversed (P:395-398,
 *     Sec. 3.3).  On a switch: m one-hop trees, GPU j roots 1/m of the
 *     data (Sec. 3.5).
 *   - The API shape follows NCCL's (the paper ships an "NCCL-compatible API",
 *     P:113): stream-ordered, asynchronous, every rank makes the same
 *     sequence of calls with the same count / dtype / op / root.
 *
 * Conventions for every entry point
 *   - Every call returns blink_result_t; BLINK_SUCCESS == 0.  On failure the
 *     comm's blink_last_error() names the offending argument / link / rank.
 *   - Buffers (sendbuf / recvbuf) are DEVICE pointers on the comm's device,
 *     owned by the caller, and must stay valid until the stream work of the
 *     call completes.  In-place iff sendbuf == recvbuf.  count is in elements.
 *   - Streams are cudaStream_t values passed as void* (NULL = legacy default
 *     stream).  Calls only enqueue work; nothing blocks the host.
 *   - The library owns its flag arrays, device tables, IPC mappings and plans;
 *     blink_destroy() synchronises the device and frees them.
 *   - One host thread per comm at a time.
 */
#ifndef BLINK_H_
#define BLINK_H_

/* Boundary vs SURVEY.md §8(b) (the planned signatures), and why it differs:
 *   blink_register                       -> blink_register_export + blink_register_connect:
 *        registration maps the PEERS' buffers (CUDA IPC), so it needs the same
 *        handle exchange as init (export/connect), not one local call.
 *   blink_config_t.slots                 -> none: partials live in the node's own recv
 *        (DESIGN §2), so there are no per-edge staging slots to size; the
 *        TMA stage ring is sized from shared memory (BLINK_SMEM_KB).
 *   blink_config_t.ctas_per_channel      -> ctas (the CTA budget per launch), split over
 *        channels in proportion to bytes x operands (a6).
 *   blink_config_t.oneshot_max_bytes     -> ll_max_bytes (the low-latency protocol), plus
 *        shallow_max_bytes (R#27) and onehop_bcast_max_bytes.
 *   cudaStream_t stream                  -> void* stream (no CUDA types in the ABI).
 *   additions: blink_reduce_scatter / blink_allgather / blink_gather (NEXT-3),
 *        blink_miad_* (NEXT-2), blink_plan_json / blink_topology_json (host-only),
 *        blink_get_stats / blink_get_trace / blink_comm_info (introspection),
 *        cfg.autotune, launch_per_rank, staging_bytes, nvls, nvls_bytes. */
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Result codes; 0..5 mirror ncclResult_t. */
typedef enum {
  BLINK_SUCCESS = 0,
  BLINK_ERR_CUDA = 1,             /* a CUDA runtime/driver call failed            */
  BLINK_ERR_SYSTEM = 2,           /* host allocation / OS failure                 */
  BLINK_ERR_INTERNAL = 3,         /* library bug                                  */
  BLINK_ERR_INVALID_ARGUMENT = 4, /* NULL, bad count/dtype/op, root out of range  */
  BLINK_ERR_INVALID_USAGE = 5,    /* call sequence or buffer contract violated    */
  BLINK_ERR_TOPOLOGY = 8,         /* disconnected allocation, bad capacity, dangling
                                     endpoint, missing reverse link for AllReduce */
  BLINK_ERR_UNSUPPORTED = 9,      /* no peer access between ranks, too many ranks,
                                     plan exceeds device-table limits             */
  BLINK_ERR_TIMEOUT = 10          /* a per-chunk flag wait exceeded cfg.timeout_s;
                                     reported by the NEXT call on that comm       */
} blink_result_t;

typedef enum { BLINK_FLOAT32 = 0, BLINK_BFLOAT16 = 1, BLINK_INT32 = 2 } blink_dtype_t;

/* "all the reduction functions supported by NCCL (e.g. min, max, etc.)".
 * SUM/PROD on floats accumulate in fp32 (bf16 widened exactly, rounded RNE once
 * per tree node); int32 wraps modulo 2^32; MIN/MAX are exact (IEEE minNum /
 * maxNum, -0 < +0). */
/* AVG (R#28): the sum along the same tree, divided by nranks at the tree root
 * before its one rounding (fp32 IEEE division; int32 truncating division). */
typedef enum { BLINK_SUM = 0, BLINK_PROD = 1, BLINK_MIN = 2, BLINK_MAX = 3, BLINK_AVG = 4 } blink_redop_t;

/* Link graph.  Nodes 0..nranks-1 are the ranks' GPUs, in rank order;
 * further nodes may be SWITCH nodes.  Each link is directed src->dst with a
 * positive bandwidth-proportional capacity; bidirectional != 0 adds the
 * reverse edge with the same capacity.  Parallel links add up.  A graph in
 * which every GPU is attached only to SWITCH nodes is planned with one-hop
 * trees. */
typedef enum { BLINK_NODE_GPU = 0, BLINK_NODE_SWITCH = 1 } blink_node_kind_t;
typedef struct {
  int src, dst;
  double capacity;
  int bidirectional;
} blink_link_t;
typedef struct {
  int num_nodes;
  const blink_node_kind_t* kinds; /* num_nodes entries; NULL = all GPU          */
  int num_links;
  const blink_link_t* links;
} blink_graph_t;

/* Configuration; pass NULL for defaults (see blink_config_default).
 *   mwu_eps        MWU approximation parameter, default 0.1
 *   ilp_gap        ILP relaxation threshold "(e.g., 5%)", default 0.05
 *   chunk_bytes    0 = size-dependent static table (a8), else fixed chunk size
 *   ctas           CTA budget per device launch; 0 = all co-resident CTAs
 *                  (occupancy x SM count)
 *   threads        threads per CTA (multiple of 32, 128..256); default 256
 *   timeout_s      flag-wait bound; expiry aborts the launch and the next call
 *                  returns BLINK_ERR_TIMEOUT; default 30
 *   onehop_bcast_max_bytes  switch graphs: Broadcast below this size uses the
 *                  single one-hop star, above it the m-1 two-level trees
 *   staging_bytes  multi-process: size of the library-owned symmetric staging
 *                  buffer used for unregistered user buffers; default 64 MiB
 *   autotune       1 = MIAD chunk-size selection across calls (
 *                  chunking never changes results).  Single process: one host
 *                  decides for every rank.  One process per GPU: rank 0
 *                  decides and publishes each call's size in its flag words,
 *                  the other ranks read it before enqueueing the call (they
 *                  wait for rank 0 to get that far).  Calls enqueued on a
 *                  stream under CUDA-graph capture use the static table
 *                  (no timing inside a capture).  Must agree across ranks.
 *                  0 = the static table (default)
 *   launch_per_rank  single-process comms only: 1 = every rank runs in its own
 *                  launch on a library-owned stream (forked from and joined
 *                  back into the rank's stream), with the cross-launch
 *                  protocol of the multi-process path (entry handshake,
 *                  per-chunk flags, exit waits) even when ranks share a
 *                  device.  Each launch gets 1/m of the device's co-resident
 *                  CTAs.  This runs the one-process-per-GPU data path
 *                  concurrently on one GPU (separate processes time-slice).
 *                  0 = ranks sharing a device are batched into one launch
 *                  (default)
 *   ll_max_bytes   switch plans: AllReduce (m one-hop trees) and the one-hop
 *                  Broadcast star up to this many bytes per rank run the
 *                  low-latency protocol (readiness flags inside the data
 *                  lines, no handshake; NEXT-2); 0 = off.
 *                  Default 256 KiB (64 KiB when one launch holds every rank,
 *                  which has no handshake to save).
 *                  On link graphs, calls of at most min(ll_max_bytes / 2,
 *                  128 KiB) on R#27's single shallow tree (see
 *                  shallow_max_bytes) run the LL protocol up and down that
 *                  tree.  Costs 64 * m * (cap) bytes of device memory per
 *                  rank, cap = ll_max_bytes / (8 m) + 8 lines (link graphs:
 *                  at least min(ll_max_bytes / 2, 128 KiB) / 8 + 8).  Must
 *                  agree across ranks
 *   shallow_max_bytes  link graphs (not switches, not multi-server): Broadcast
 *                  and AllReduce calls of at most this many bytes per rank run
 *                  on ONE minimum-depth (BFS) tree -- from the root, or from
 *                  the graph's centre for AllReduce -- instead of the packed
 *                  trees: small calls are latency-bound and every hop waits
 *                  for a whole chunk (depth-1 trees on the
 *                  switch).  Default 256 KiB; 0 = always packed.
 *                  Must agree across ranks
 *   nvls           NEXT-1: 1 = run the switch's one-hop trees inside the
 *                  NVSwitch (multicast objects: multimem.ld_reduce reduces
 *                  slice j of every rank in the switch, multimem.st writes the
 *                  result to every rank; Broadcast = the root's multimem.st)
 *                  for AllReduce SUM (f32, bf16, int32) and Broadcast above
 *                  the LL sizes, 16-byte-aligned buffers.  Needs one rank per
 *                  device on >= 2 multicast-capable GPUs (multi-process: a
 *                  FABRIC handle, or without FABRIC support a POSIX fd that the
 *                  ranks duplicate from rank 0's process with pidfd_getfd, so
 *                  one node and ptrace access); otherwise the P2P stars run and blink_get_plan's
 *                  "nvls" says why.  Float sums then follow the switch's
 *                  order, not ascending ranks (within the north_star
 *                  tolerance).  0 = off (default).  Must agree across ranks
 *   nvls_bytes     multicast-bound buffer per rank (calls run in pieces of
 *                  this size); default 64 MiB */
typedef struct {
  double mwu_eps;
  double ilp_gap;
  size_t chunk_bytes;
  int ctas;
  int threads;
  double timeout_s;
  size_t onehop_bcast_max_bytes;
  size_t staging_bytes;
  int autotune;
  int launch_per_rank;
  size_t ll_max_bytes;
  size_t shallow_max_bytes;
  int nvls;
  size_t nvls_bytes;
} blink_config_t;

/* MIAD controller: "initialize the chunk size with a small value
 * and increase the chunk size by a multiplicative factor as long as the
 * measured throughput is increasing.  If the throughput decreases we additively
 * decrease the chunk size until we reach a steady state."  init = 1 MiB,
 * factor 2, additive step = init, "increasing" = more than 1% better.
 * blink_miad_init sets the state; each blink_miad_step feeds the throughput
 * measured with state->chunk and returns the chunk size to use next.  Pure host
 * function (the runtime drives it from CUDA-event timings when cfg.autotune). */
typedef struct {
  size_t chunk, best, init, step, min_chunk, max_chunk;
  double last_thr, best_thr, tol;
  int phase; /* 0 multiplicative increase, 1 additive decrease, 2 steady */
  int iters;
} blink_miad_t;
void blink_miad_init(blink_miad_t* st, size_t init, size_t min_chunk, size_t max_chunk);
size_t blink_miad_step(blink_miad_t* st, double throughput);

void blink_config_default(blink_config_t* cfg);

typedef struct blink_comm* blink_comm_t;

/* ---------------------------------------------------------------- control plane
 * Host-only planning (no GPU needed): TreeGen for a graph plus the
 * split and chunking of `count` elements.  Writes a JSON document
 * {"coll","root","count","esize","rate":[num,den],"trees":[{"root","parent":[],
 * "weight":[num,den],"depth","lo","hi","chunk","nchunks"}]} (lo/hi/chunk in
 * elements).  *json_bytes is in/out: capacity in, required size (incl. NUL)
 * out; BLINK_ERR_INVALID_ARGUMENT if the capacity is too small.
 * graph == NULL means the NVSwitch model (all ranks behind one switch).
 * `is_allreduce` selects the collective: 0 Broadcast, 1 AllReduce, and (NEXT-3)
 * 2 ReduceScatter, 3 AllGather, 4 Gather, whose trees cover one block each. */
blink_result_t blink_plan_json(const blink_graph_t* graph, int nranks, const blink_config_t* cfg,
                               int is_allreduce, int root, size_t count, blink_dtype_t dtype,
                               char* json, size_t* json_bytes);

/* ---------------------------------------------------------------- init
 * Single-process init of ndev ranks (like ncclCommInitAll).  devs[i] is rank
 * i's CUDA device; devices may repeat, in which case the ranks sharing a
 * device are "virtual ranks" whose buffers all live in that GPU's HBM and
 * whose calls are batched into one launch (needed on a 1-GPU box).  Ranks on
 * distinct devices need peer access (enabled here).  graph == NULL probes:
 * all-pairs peer access => switch model, else BLINK_ERR_UNSUPPORTED. */
blink_result_t blink_init_all(blink_comm_t* comms, int ndev, const int* devs,
                              const blink_graph_t* graph, const blink_config_t* cfg);

/* Multi-process init (one GPU per process).  The handle exchange is the
 * caller's: blink_export_handle() fills a blob (<= 512 bytes), the caller
 * all-gathers the nranks blobs in rank order (e.g. torch.distributed over
 * gloo) and passes them to blink_connect(), which maps the peers' flag arrays
 * and staging buffers (CUDA IPC over NVLink) and builds the plans. */
blink_result_t blink_init(blink_comm_t* comm, int nranks, int rank, int cuda_device,
                          const blink_graph_t* graph, const blink_config_t* cfg);
blink_result_t blink_export_handle(blink_comm_t comm, void* blob, size_t* blob_bytes);
blink_result_t blink_connect(blink_comm_t comm, const void* all_blobs, size_t blob_bytes);

/* Symmetric buffer registration (multi-process zero-copy).  Collective: every
 * rank registers its own buffer of the same size in the same order, exports a
 * blob, all-gathers the blobs (caller's channel) and connects.  Registered
 * buffers are used in place; unregistered ones go through the library staging
 * buffer; collectives on a registered buffer must use the same byte offset
 * into it on every rank.  No-ops (SUCCESS) on single-process comms.
 *   cudaMalloc memory (incl. PyTorch's caching allocator): a CUDA IPC handle
 *   of the allocation plus the offset.  VMM memory (e.g. PyTorch
 *   expandable_segments): every physical chunk the buffer touches is exported
 *   as a POSIX fd; peers duplicate the fds (pidfd_getfd: needs ptrace access
 *   to the exporter, e.g. same user with ptrace_scope 0, or CAP_SYS_PTRACE)
 *   and map the chunks back to back.  The exporter keeps the fds until
 *   blink_destroy.
 * blink_register_export with blob == NULL only reports the blob size in
 * *blob_bytes.  Errors: UNSUPPORTED (neither kind of memory, or more than
 * 128 VMM chunks), SYSTEM (pidfd failures), CUDA. */
blink_result_t blink_register_export(blink_comm_t comm, void* buf, size_t bytes, void* blob,
                                     size_t* blob_bytes);
blink_result_t blink_register_connect(blink_comm_t comm, void* buf, const void* all_blobs,
                                      size_t blob_bytes);

/* ---------------------------------------------------------------- collectives
 * Broadcast `count` elements of root's sendbuf into every rank's recvbuf
 * (P:477-478).  sendbuf is read on the root only (may be NULL elsewhere). */
blink_result_t blink_broadcast(blink_comm_t comm, const void* sendbuf, void* recvbuf, size_t count,
                               blink_dtype_t dtype, int root, void* stream);
/* AllReduce of `count` elements.  Every rank's recvbuf
 * receives the same result, computed along the packed trees in the fixed
 * per-node operand order (ascending rank, R#12). */
blink_result_t blink_allreduce(blink_comm_t comm, const void* sendbuf, void* recvbuf, size_t count,
                               blink_dtype_t dtype, blink_redop_t op, void* stream);

/* ReduceScatter (NEXT-3: the reduce half of AllReduce).
 * sendbuf holds nranks blocks of recvcount elements; rank j's recvbuf
 * (recvcount elements) receives block j reduced over all ranks.  Switch: the
 * one-hop star rooted at j, ascending rank order.  Link graphs: a
 * minimum-depth spanning tree rooted at j over bidirectional links, each node
 * combining its own block with its children's partials in ascending rank
 * order (R#12); inner ranks relay partials through a library-owned area
 * (single process: scratch; multi-process: the staging buffer's second
 * half).  Multi-server graphs: BLINK_ERR_UNSUPPORTED. */
blink_result_t blink_reduce_scatter(blink_comm_t comm, const void* sendbuf, void* recvbuf,
                                    size_t recvcount, blink_dtype_t dtype, blink_redop_t op,
                                    void* stream);
/* AllGather (NEXT-3: "AllReduce without using a reduction function").
 * Every rank's sendcount elements land at block `rank` of every recvbuf
 * (nranks*sendcount elements).  In place iff sendbuf == recvbuf + rank*sendcount.
 * Switch: block j is pushed by root j along its one-hop star.  Link graphs:
 * block j is broadcast down a minimum-depth arborescence rooted at j (the m
 * arborescences spread over the links); multi-server graphs are unsupported. */
blink_result_t blink_allgather(blink_comm_t comm, const void* sendbuf, void* recvbuf,
                               size_t sendcount, blink_dtype_t dtype, void* stream);

/* Gather (NEXT-3: "Gather is the inverse of Broadcast").  Every rank's
 * sendcount elements land at block `rank` of the root's recvbuf
 * (nranks*sendcount elements); recvbuf is unused (may be NULL) on other
 * ranks.  Switch: rank j's block travels the single edge j -> root (one-hop
 * trees).  Link graphs: block j travels j's path to the root in the root's
 * minimum-depth Broadcast tree, reversed (intermediate ranks forward it; in
 * single-process comms a rank with recvbuf == NULL forwards through a
 * library-owned scratch buffer). */
blink_result_t blink_gather(blink_comm_t comm, const void* sendbuf, void* recvbuf,
                            size_t sendcount, blink_dtype_t dtype, int root, void* stream);

/* Eq. 8 (Sec. 3.4 "Handling hybrid communication"): the data
 * split between PCIe trees and NVLink trees that equalises
 * T_PCIe + T_dpa = T_NVL:  D_PCIe = D_total BW_PCIe / (BW_PCIe + BW_NVL)
 * - T_dpa BW_PCIe BW_NVL / (BW_PCIe + BW_NVL), D_NVL = D_total - D_PCIe.
 * Bandwidths in bytes/s, T_dpa (cudaDeviceDisablePeerAccess latency) in s.
 * D_PCIe is clamped to [0, D_total] and rounded down to 16 bytes.  Host-only
 * planning (the hybrid data path is out of scope on B200).  Errors:
 * INVALID_ARGUMENT for NULL outputs, nonpositive bandwidths, negative T_dpa. */
blink_result_t blink_hybrid_split(size_t d_total, double bw_pcie, double bw_nvl, double t_dpa,
                                  size_t* d_pcie, size_t* d_nvl);

/* ---------------------------------------------------------------- topology probe
 * "Blink probes the set of links available ... and builds a topology with
 * appropriate link capacities" (Sec. 1; Sec. 2.3).  For the GPUs
 * named by their PCI bus ids (cudaDeviceGetPCIBusId format), reads every
 * active NVLink port from NVML (loaded at run time) and writes
 * {"kind": "virtual"|"nvswitch"|"nvlink"|"pcie", "switch_ports": [per GPU],
 *  "links": [[u, v, ports], ...], "note": "..."}.  "nvlink" graphs (direct
 * GPU-GPU links; capacity = parallel links) are packed (Sec. 3.2); the other
 * kinds use the one-hop switch model.  blink_init / blink_init_all run this
 * probe when graph == NULL, and blink_get_plan reports it under "topology".
 * Host only; BLINK_FAKE_NVML=<file> substitutes a port table ("<bus id>
 * <port> <remote bus id | switch>" per line).  json/json_bytes as for
 * blink_plan_json.  Errors: INVALID_ARGUMENT (NULL, bad bus id, small
 * buffer), UNSUPPORTED (ndev outside 1..16), SYSTEM (unreadable fake table).
 * Without NVML the kind is "pcie" and "note" says why. */
blink_result_t blink_topology_json(int ndev, const char* const* bus_ids, char* json, size_t* json_bytes);

/* ---------------------------------------------------------------- introspection
 * Same JSON as blink_plan_json, for the plan this comm would run, plus "ctas"
 * (CTAs of this rank's launch). */
blink_result_t blink_get_plan(blink_comm_t comm, int is_allreduce, int root, size_t count,
                              blink_dtype_t dtype, char* json, size_t* json_bytes);
/* Launch statistics of the most recent call that reached the device:
 * kernels launched by it, CTAs, chunks. */
typedef struct {
  int64_t launches;      /* cumulative kernel launches by this comm's device batch */
  int last_ctas;
  int last_chunks;
  int last_trees;
  int64_t last_chunk_bytes;  /* chunk size of tree 0 in the last launch (MIAD trace) */
  int last_steal_channels;   /* channels CTAs may join in the last launch (work stealing; 0 = off) */
} blink_stats_t;
blink_result_t blink_get_stats(blink_comm_t comm, blink_stats_t* stats);
/* Device-side trace of the last launch on this comm's device when the
 * environment variable BLINK_TRACE is set (single-process comms): 16 %globaltimer
 * stamps (ns) per CTA -- start, epoch read, entry handshake done, first TMA
 * load, first bulk store, last stores complete, end of work, after the epoch
 * update; then the hop's parts in the CTA's last segment: 8 producer has the
 * first chunk's inputs (flags acquired), 9 store thread sees the first stage
 * full, 10 store thread sees the end of the stream, 11 stores drained, 12
 * chunk signals published, 13-15 spare (0 where a CTA has no such event).
 * *n_words in/out like
 * blink_plan_json; synchronous copy.  *n_words = 0 when tracing is off. */
blink_result_t blink_get_trace(blink_comm_t comm, uint64_t* out, size_t* n_words);
blink_result_t blink_comm_info(blink_comm_t comm, int* nranks, int* rank, int* device);

blink_result_t blink_destroy(blink_comm_t comm);
const char* blink_result_string(blink_result_t r);
const char* blink_last_error(blink_comm_t comm); /* comm may be NULL: last global error */

#ifdef __cplusplus
}
#endif
#endif /* BLINK_H_ */
