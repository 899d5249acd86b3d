// qt_internal.h -- kernel argument blocks and launchers shared by
// qt_kernels.cu (device) and qt_capi.cu (host runtime).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "qt_layout.h"

namespace qt {

// The caller's current CUDA device (0 when the runtime has none to report).
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    d = 0;
  }
  return d;
}

// Saves the current device on entry to a C-ABI call and restores it on exit,
// so no entry point (nor a plan destructor it triggers) changes the caller's
// device. No-op when there is no device.
struct DeviceRestore {
  int dev = -1;
  DeviceRestore() {
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      dev = -1;
    }
  }
  ~DeviceRestore() {
    if (dev >= 0) cudaSetDevice(dev);
  }
  DeviceRestore(const DeviceRestore&) = delete;
  DeviceRestore& operator=(const DeviceRestore&) = delete;
};

// Normal-source parameters (see Source<> in qt_device.cuh).
struct SrcArgs {
  uint32_t mrg_seed[6];
  uint64_t lcg_seed;
  uint64_t seed;
  const uint32_t* mrg_table;
  const unsigned long long* lcg_table;
  const double* normals;
  uint64_t normals_first;
  uint64_t draws;
  uint32_t per_unit;
};

// An uncertified path of the certified 1-D kernels (k_paths_fast, k_paths_x<CERT>),
// replayed exactly by k_replay.
struct AmbEntry {
  unsigned long long key;  // (path << 16) | first uncertified layer
  uint32_t st[6];          // MRG32k3a state at the path's first draw
};
static_assert(sizeof(AmbEntry) == 32, "AmbEntry is 32 bytes");

struct PathArgs {
  SrcArgs src;
  const uint8_t* tables;      // layer tables, concatenated, 16-byte aligned
  const uint32_t* tab_off;    // [n] byte offset of layer k's table (index k-1)
  const uint32_t* tab_bytes;  // [n]
  unsigned long long* joint;
  uint64_t first;             // first path of the window
  uint64_t q, rem;            // window split over T threads: q each, +1 for the first rem
  uint32_t n;
  uint32_t buf_bytes;         // staging buffer size (max table bytes)
  uint32_t resident_bytes;    // sum of table bytes (resident mode)
  uint32_t stages;            // shared-memory ring depth (power of 2, <= 8)
  uint32_t layers_per_stage;  // k_paths_x: layer tables per pipeline stage (1 or 2)
  uint32_t probe_nored;       // diagnostics only (QT_PROBE_NORED): skip the count REDs
  const uint8_t* xtables;     // k_paths_x: the d = 1 tables with Thr[] replaced by
                              // threshold pairs {t_c, t_c+1} (same offsets; counts are
                              // in sorted-cell space, see launch_permute_add)
  // k_paths_x<CERT>: the uncertified paths' replay list and the original-index
  // counts an overflowing list is replayed into inline
  AmbEntry* amb;
  unsigned long long* stats;  // [0] list entries of this launch, [1], [2] as FastArgs
  uint64_t amb_cap;
  unsigned long long* ojoint;
  uint32_t back[18];          // (J^D)^-1: path end state -> path start state
  // k_paths_x: the first transition (x0 -> layer 1: every path lands in one of
  // N_1 cells of a single row) counted in a per-CTA shared-memory histogram of
  // n1 u32 at byte offset hist1_off of the dynamic smem, flushed once per CTA;
  // n1 = 0: one RED per path like the other layers
  uint32_t n1;
  uint32_t hist1_off;
};

constexpr int kPathConsumers = 256;  // consumer threads per k_paths CTA
#ifndef QT_X_MINB  // k_paths_x: resident CTAs per SM the register allocation must allow
#define QT_X_MINB 1
#endif
#ifndef QT_X_THREADS
#define QT_X_THREADS 256
#endif
constexpr int kXThreads = QT_X_THREADS;  // k_paths_x CTA: warps in layer lockstep

struct FastArgs {
  PathArgs p;
  AmbEntry* amb;              // ambiguous paths
  unsigned long long* stats;  // [0] entries of this launch, [1] replayed (cumulative),
                              // [2] replayed inline on list overflow (cumulative)
  uint64_t cap;               // capacity of amb
  const uint8_t* ftables;     // fast-path tables (FastHdr + FRec[]), concatenated
  const uint32_t* ftab_off;   // [n]
  const uint32_t* ftab_bytes; // [n]
  uint32_t fbuf_bytes;        // ring stage size (max fast table)
  uint32_t fresident_bytes;   // sum of fast tables (resident mode)
  uint32_t fstages;           // prefetch depth (stages of fbuf_bytes)
  uint32_t back[18];          // (J^D)^-1 mod m1 | mod m2: path end -> path start
  uint32_t probe_nored;       // diagnostics only (QT_PROBE_NORED): skip the count REDs
  unsigned long long* sjoint; // certified counts, SORTED-cell space (launch_permute_add maps
                              // them to p.joint); replays count into p.joint directly
  uint32_t flayers;           // layers per ring stage (1 or 2)
};

// d >= 2 FP32-scan path kernel (qt_scan.cu)
struct ScanArgs {
  PathArgs p;                 // exact tables (p.tables: FP64 points, global) + joint + window
  const uint8_t* stables;     // scan tables (ScanHdr + FP32 pairs), concatenated
  const uint32_t* stab_off;   // [n]
  const uint32_t* stab_bytes; // [n]
  uint32_t sbuf_bytes;        // stage size (max scan table)
  uint32_t sresident_bytes;   // sum of scan tables (resident mode)
  uint32_t sstages;           // prefetch depth
};

struct Alg3Args {
  SrcArgs src;
  const uint8_t* tables;
  const uint32_t* tab_off;
  const uint32_t* tab_bytes;
  unsigned long long* joint;
  uint64_t M;             // samples per layer
  uint64_t first, count;  // unit window within [0, n M)
  uint32_t n;
  uint32_t buf_bytes;
  uint32_t probe_nored;   // diagnostics only (QT_PROBE_NORED): skip the count REDs
  const uint8_t* xtables;  // k_alg3_x: threshold-pair tables (see PathArgs::xtables)
  // k_alg3_x<CERT>: uncertified samples (key = unit << 16 | k) for k_replay3, the
  // original-index counts they and an overflowing list are replayed into, and
  // (J^2)^-1 (the state after a sample's pair -> the state before it)
  AmbEntry* amb;
  unsigned long long* stats;
  uint64_t amb_cap;
  unsigned long long* ojoint;
  uint32_t back2[18];
  // k_alg3_x<PRIV>: bytes of the CTA's shared-memory count tile (n_{k-1} x n_k
  // u32 counters after the two table buffers), flushed to `joint` at the end
  uint32_t priv_bytes;
};

// d >= 2 cell-list path kernels (qt_cell.cu): exact tables (FP64 points) and
// the cell-list tables, both read from global memory (L2-resident)
struct CellArgs {
  PathArgs p;
  const CellHdr* chdr;        // [n] layer k's header at index k-1
  const uint32_t* cstart;     // bucket list starts, all layers (+ a final end)
  const uint16_t* clist;      // candidate point indices, ascending per bucket
  const uint4* crec;          // per bucket: up to 7 candidates inline (x: n | c0 << 16,
                              // y..w: c1..c6), or n = 0xFFFF: y = list start, z = count
};
struct Alg3CellArgs {
  Alg3Args a;
  const CellHdr* chdr;
  const uint32_t* cstart;
  const uint16_t* clist;
  const uint4* crec;
};
// Builds the cell lists of n layers on the current device (synchronous):
// hdr[n] (host) geometry with start_off set, npts[n] = N_k, the FP64 points of
// layer k at tables + pts_off[k-1]. Allocates *d_hdr, *d_start, *d_list.
cudaError_t build_cell_lists(int dim, int n, const CellHdr* hdr, const uint64_t* npts,
                             const uint8_t* tables, const uint64_t* pts_off, CellHdr** d_hdr,
                             uint32_t** d_start, uint16_t** d_list, uint4** d_rec,
                             uint64_t* total);

struct FinalizeArgs {
  const uint64_t* rows;      // [n] N_{t}
  const uint64_t* cols;      // [n] N_{t+1}
  const uint64_t* joff;      // [n] joint offset of transition t
  const uint64_t* voff_row;  // [n] visits offset of layer t
  const uint64_t* voff_col;  // [n] visits offset of layer t+1
};

// Alg III with the FP32 scan projection (d >= 2, qt_scan.cu)
struct Alg3ScanArgs {
  Alg3Args a;                 // a.tables: exact tables (FP64 points, global; decisions)
  const uint8_t* stables;     // scan tables (ScanHdr + FP32 pairs), concatenated
  const uint32_t* stab_off;   // [n]
  const uint32_t* stab_bytes; // [n]
  uint32_t sbuf_bytes;        // max scan table
};

// shared error text / launch counter (defined in qt_capi.cu)
void note_error(const std::string& msg);
void note_launches(uint64_t n);
// pageable host <-> device copy staged through pinned buffers (qt_capi.cu)
cudaError_t staged_copy(void* dst, const void* src, size_t bytes, bool to_device,
                        cudaStream_t st);

cudaError_t launch_paths(int kind, int src, bool resident, const PathArgs& a, uint32_t blocks,
                         size_t smem, cudaStream_t st);
int paths_blocks_per_sm(int kind, int src, bool resident, size_t smem);
cudaError_t launch_paths_fast(int kind, bool resident, int P, const FastArgs& a, uint32_t blocks,
                              size_t smem, uint32_t replay_blocks, cudaStream_t st);
int paths_fast_blocks_per_sm(int kind, bool resident, int P, size_t smem);
cudaError_t launch_fast_bounds_check(unsigned int* out, cudaStream_t st);
cudaError_t launch_math_checksum(int domain, unsigned long long* out, cudaStream_t st);
cudaError_t launch_serial_normals(const SrcArgs& a, uint64_t first, uint64_t count, double* out,
                                  cudaStream_t st);
cudaError_t launch_lloyd_update(const double* X, const unsigned long long* cell, uint64_t M,
                                uint64_t N, int d, double* centers, double* d2, uint32_t* key,
                                uint32_t* idx, uint32_t* key2, uint32_t* idx2, uint32_t* counts,
                                uint32_t* offs, void* tmp, size_t tmp_bytes, cudaStream_t st);
size_t lloyd_tmp_bytes(uint64_t M, uint64_t N);
cudaError_t launch_pi(int engine, int skip, const SrcArgs& a, uint64_t samples, uint64_t streams,
                      unsigned long long* inside, cudaStream_t st);
cudaError_t launch_sum_u64(const unsigned long long* v, uint64_t n, unsigned long long* out,
                           cudaStream_t st);
cudaError_t launch_paths_x(int kind, bool resident, int P, bool cert, const PathArgs& a,
                           uint32_t blocks, size_t smem, cudaStream_t st, int* bps);
cudaError_t launch_replay(int kind, const FastArgs& f, uint32_t blocks, cudaStream_t st);
cudaError_t launch_replay3(int kind, const Alg3Args& a, uint32_t blocks, cudaStream_t st);
cudaError_t launch_apx_bounds_check(unsigned long long* out, cudaStream_t st);
// joint[t][orig_t[a] N_{t+1} + orig_{t+1}[b]] += sjoint[t][a N_{t+1} + b] for every
// layer t (sorted-cell counts of k_paths_x -> the reference's original indices);
// fin = the finalize table (rows, cols, joff, voff_row, voff_col; 5 x n), orig
// indexed by voff.
// estimate -> price without the pi round trip (qt_bdp.cu): visits / pi are
// device arrays on the current device; phi and the outputs are host arrays.
// Failures throw BdpError {qt_status code, message}.
struct BdpError {
  int code;
  std::string msg;
};
void bdp_stopping_device(int32_t layers, const uint64_t* sizes, const uint64_t* d_visits,
                         const double* d_pi, const double* phi, double* value, uint8_t* exercise,
                         double* price);
void bdp_swing_device(int32_t layers, const uint64_t* sizes, const uint64_t* d_visits,
                      const double* d_pi, const double* phi, int32_t qmin, int32_t qmax,
                      double* price, double* value_all, uint8_t* take_all);

cudaError_t launch_permute_add(const unsigned long long* sjoint, unsigned long long* joint,
                               const uint64_t* fin, const uint32_t* orig, uint32_t n,
                               uint64_t max_elems, cudaStream_t st);
cudaError_t launch_paths_scan(int kind, int src, bool resident, int P, const ScanArgs& a,
                              uint32_t blocks, size_t smem, cudaStream_t st);
int paths_scan_blocks_per_sm(int kind, int src, bool resident, int P, size_t smem);
cudaError_t launch_paths_cell(int kind, int src, int P, const CellArgs& a, uint32_t blocks,
                              cudaStream_t st);
int paths_cell_blocks_per_sm(int kind, int src, int P);
cudaError_t launch_alg3_cell(int kind, int src, const Alg3CellArgs& a, uint32_t slices,
                             cudaStream_t st);
cudaError_t launch_alg3_scan(int kind, int src, const Alg3ScanArgs& a, uint32_t slices,
                             size_t smem, cudaStream_t st);
cudaError_t launch_nearest_scan(int dim, const uint8_t* stable, uint32_t sbytes,
                                const uint8_t* xtable, const double* q, uint64_t nq,
                                unsigned long long* out, cudaStream_t st);
cudaError_t launch_alg3(int kind, int src, const Alg3Args& a, uint32_t slices, size_t smem,
                        cudaStream_t st);
cudaError_t launch_alg3_x(int kind, int P, bool cert, const Alg3Args& a, uint32_t slices,
                          size_t smem, cudaStream_t st);
cudaError_t launch_gmem(int kind, int src, bool alg3, const PathArgs& pa, const Alg3Args& aa,
                        uint32_t blocks, cudaStream_t st);
cudaError_t launch_finalize(bool alg3, const unsigned long long* joint, unsigned long long* visits,
                            double* pi, uint64_t samples, const FinalizeArgs& f, uint32_t n,
                            uint64_t max_cols, uint64_t max_rows, uint64_t max_elems,
                            cudaStream_t st, int* launches);
cudaError_t launch_nearest(int dim, const uint8_t* table, uint32_t bytes, const double* q,
                           uint64_t nq, unsigned long long* out, cudaStream_t st);
cudaError_t launch_path_normals(int src, const SrcArgs& a, uint64_t first, uint64_t count,
                                double* out, cudaStream_t st);
cudaError_t launch_uniforms(int src, const SrcArgs& a, uint64_t offset, uint64_t count,
                            double* out, cudaStream_t st);

}  // namespace qt
