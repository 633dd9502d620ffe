// engine.cu — the B200 program-counter VM (paper Alg. 2 / reference pc_vm.py) and its C ABI.
//
// Two engines share the per-lane semantics of lsb_vm.cuh (exec_block):
//
//   vm_cta_kernel  — "exact" / "cta": one CTA is one autobatching group of up
//                    to 1024 lanes (one thread per lane). Each step the CTA
//                    reduces its live lanes' program counters (warp min /
//                    __match_any_sync histogram + shared-memory combine),
//                    selects one block, and the threads at that block run it.
//                    With one group this reproduces the reference's global
//                    min-pc schedule step for step (pc_vm.py:304-332).
//   vm_warp_kernel — "warp": the throughput engine. Every warp is its own
//                    32-lane group scheduled by warp votes, with no CTA
//                    barriers; target gradients run warp-cooperatively on the
//                    fp64 tensor pipe (DMMA) and recognised leapfrog functions
//                    run as fused superblocks. Lanes refill from a chain queue.
//
// Both kernels are persistent and resumable: all machine state lives in HBM
// (per-group workspaces), so a launch may stop after any step. Faults are
// reported as the lowest (op position, lane) of the faulting step like
// reference runtime.py:462-507, and stop the machine (no rollback).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lockstep_b200.h"
#include "lsb_vm.cuh"

// A program-specialised build (codegen.py) replaces the warp engine's block
// interpreter with generated straight-line block functions.
#ifdef LSB_GENERATED
#include LSB_GENERATED
#else
#define LSB_WARP_EXEC(...) exec_block<true>(__VA_ARGS__)
#endif

using namespace lsbvm;
using lsb::as_f64;
using lsb::f64_bits;

namespace {

struct CtaShared {
  int pick;
  unsigned pick_key;
  int count;
  unsigned long long fault_key;
  int warp_val[kMaxLanes / 32];
  int warp_cnt[kMaxLanes / 32];
};

__global__ void __launch_bounds__(kMaxLanes) vm_cta_kernel(const __grid_constant__ VMArgs a) {
#ifndef LSB_GENERATED  // program-specialised libraries run the warp engine only
  extern __shared__ int s_hist[];  // [n_blocks + 1]
  __shared__ CtaShared sh;
  const int g = blockIdx.x;
  const int t = threadIdx.x;
  const int L = a.lanes;
  const int lane_id = t & 31, warp = t >> 5, nwarps = (L + 31) >> 5;
  const Lane ln{a.ws + (size_t)g * a.group_rows * L, a.sp + (size_t)g * a.n_sp_rows * L,
                a.pcs + (size_t)g * (a.depth + 1) * L, t, L};
  int* pc_sp = &ln.sp_row(a.n_sp_rows - 1);
  long long* my_chain = a.chain_of + (size_t)g * L + t;
  long long steps = a.group_steps[g];
  long long* bsteps = a.blk_steps + (size_t)g * a.n_blocks;
  long long* bactive = a.blk_active + (size_t)g * a.n_blocks;
  unsigned long long useful = 0, launched = 0;
  if (a.group_done[g]) return;

  for (;;) {
    if (a.refill && *my_chain == -1) {
      const unsigned long long c = atomicAdd(a.next_chain, 1ull);
      if ((long long)c < a.z) {
        *my_chain = (long long)c;
        init_lane(a, ln, (long long)c);
      } else {
        *my_chain = -2;
      }
    }
    const int pc = *my_chain >= 0 ? ln.pcs[(*pc_sp - 1) * L + t] : a.halt;
    if (t == 0) sh.fault_key = ~0ull;
    if (a.sched == LS_SCHED_MOST_POPULATED) {
      for (int b = t; b <= a.n_blocks; b += L) s_hist[b] = 0;
      __syncthreads();
      const unsigned peers = __match_any_sync(kFull, pc);
      if (pc != a.halt && lane_id == __ffs(peers) - 1) atomicAdd(&s_hist[pc], __popc(peers));
      __syncthreads();
      int best = -1, best_b = a.halt;
      for (int b = t; b < a.n_blocks; b += L) {
        const int c = s_hist[b];
        if (c > best) { best = c; best_b = b; }
      }
      unsigned long long key = best > 0 ? (((unsigned long long)(unsigned)best) << 32) |
                                              (unsigned)(0x7fffffff - best_b) : 0ull;
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(kFull, key, o);
        key = other > key ? other : key;
      }
      if (lane_id == 0) {
        sh.warp_val[warp] = (int)(key >> 32);
        sh.warp_cnt[warp] = (int)(0x7fffffff - (int)(key & 0xffffffffu));
      }
      __syncthreads();
      if (t == 0) {
        int bc = 0, bb = a.halt;
        for (int w2 = 0; w2 < nwarps; ++w2) {
          const int c = sh.warp_val[w2], b = sh.warp_cnt[w2];
          if (c > bc || (c == bc && c > 0 && b < bb)) { bc = c; bb = b; }
        }
        sh.pick = bc > 0 ? bb : a.halt;
        sh.count = bc;
      }
      __syncthreads();
    } else {
      // keyed rules (min_pc, priority, local): least key over the group's live lanes
      const unsigned key = pc == a.halt ? 0xffffffffu : lane_key(a, pc, *pc_sp);
      const unsigned m = __reduce_min_sync(kFull, key);
      if (lane_id == 0) sh.warp_val[warp] = (int)m;
      __syncthreads();
      if (t == 0) {
        unsigned mm = 0xffffffffu;
        for (int w2 = 0; w2 < nwarps; ++w2) mm = min(mm, (unsigned)sh.warp_val[w2]);
        sh.pick = mm == 0xffffffffu ? a.halt : (int)(mm & 0xffffu);
        sh.pick_key = mm;
      }
      __syncthreads();
      const unsigned bal = __ballot_sync(kFull, key == sh.pick_key && pc != a.halt);
      if (lane_id == 0) sh.warp_cnt[warp] = __popc(bal);
      __syncthreads();
      if (t == 0) {
        int c = 0;
        for (int w2 = 0; w2 < nwarps; ++w2) c += sh.warp_cnt[w2];
        sh.count = c;
      }
      __syncthreads();
    }
    const int b = sh.pick;
    if (b == a.halt) {
      if (t == 0) a.group_done[g] = 1;
      break;
    }
    if (*(volatile int*)a.abort_flag) break;
    if (a.max_steps >= 0 && steps >= a.max_steps) {
      if (t == 0) a.paused[0] = 1;
      break;
    }
    if (a.trace_block != nullptr && *a.trace_n >= a.trace_cap) {  // host drains and resumes
      if (t == 0) a.paused[1] = 1;
      break;
    }
    const bool active = pc == b && (a.sched == LS_SCHED_MOST_POPULATED || lane_key(a, pc, *pc_sp) == sh.pick_key);
    if (active && a.lane_trace != nullptr) lane_trace_put(a, *my_chain, b);
    StepFault f;
    const bool halted_now = exec_block<false>(a, ln, b, active, *my_chain, f, nullptr);
    if (f.pos) atomicMin(&sh.fault_key, ((unsigned long long)(f.pos - 1) << 32) | (unsigned)t);
    __syncthreads();
    if (sh.fault_key != ~0ull) {
      if ((unsigned)(sh.fault_key & 0xffffffffu) == (unsigned)t && f.pos &&
          (unsigned)(f.pos - 1) == (unsigned)(sh.fault_key >> 32)) {
        FaultRec& fr = a.fault[g];  // one slot per group: the host picks the lowest chain
        fr.key = sh.fault_key;
        fr.kind = f.kind;
        fr.var = f.var;
        fr.block = b;
        fr.detail = f.detail;
        fr.chain = *my_chain;
        __threadfence();
        atomicExch(a.abort_flag, 1);
      }
      steps++;
      break;
    }
    if (halted_now) {
      write_output(a, ln, *my_chain);
      if (a.refill) *my_chain = -1;
    }
    if (t == 0) {
      if (a.trace_block != nullptr) {
        const long long n = *a.trace_n;
        a.trace_block[n] = b;
        a.trace_active[n] = sh.count;
        *a.trace_n = n + 1;
      }
      const int grads = a.blocks[b].grads;
      bsteps[b] += 1;
      bactive[b] += sh.count;
      useful += (unsigned long long)sh.count * (unsigned long long)grads;
      launched += (unsigned long long)L * (unsigned long long)grads;
    }
    ++steps;
    __syncthreads();
  }
  if (t == 0) {
    a.group_steps[g] = steps;
    if (useful) atomicAdd(a.useful, useful);
    if (launched) atomicAdd(a.launched, launched);
  }
#endif
}

// up to LSB_WARPS_MAX warps per CTA (one CTA per SM): 16 -> 128 registers per thread (the
// fp64 DMMA superblock keeps the momentum in registers); builds for the fp32 arm may trade
// registers for more resident warps (24 -> 85 registers), since its superblock works in TMEM
#ifndef LSB_WARPS_MAX
#define LSB_WARPS_MAX 16
#endif
constexpr int kWarpCtaMax = LSB_WARPS_MAX;
static_assert(kWarpCtaMax <= 32, "at most 8 warpgroups per CTA");

// One warp's 32-lane group: the step loop of the warp engine. Warps step independently; in
// the fp32 arm the warps of a warpgroup meet only at the tensor-core superblock
// (wg_rendezvous), which then runs all their chains at once.
__device__ __forceinline__ void warp_group_run(const VMArgs& a, double* lf_smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = blockIdx.x * (blockDim.x >> 5) + wid;
  constexpr int L = 32;
  const Lane ln{a.ws + (size_t)g * a.group_rows * L, a.sp + (size_t)g * a.n_sp_rows * L,
                a.pcs + (size_t)g * (a.depth + 1) * L, lane, L};
  double* my_smem = lf_smem + a.stage_doubles + (size_t)wid * a.lf_smem_per_warp;
  int* pc_sp = &ln.sp_row(a.n_sp_rows - 1);
  long long* my_chain = a.chain_of + (size_t)g * L + lane;
  long long steps = a.group_steps[g];
  long long* bsteps = a.blk_steps + (size_t)g * a.n_blocks;
  long long* bactive = a.blk_active + (size_t)g * a.n_blocks;
#if LSB_BLOCK_PROFILE
  long long* bcycles = a.blk_cycles + (size_t)g * a.n_blocks;
#endif
  unsigned long long useful = 0, launched = 0;
  // the lane's chain id lives in a register; chain_of is updated whenever it changes
  long long chain = *my_chain;
#ifdef LSB_GENERATED
  // generated blocks keep the current pc and the pc-stack pointer in registers; memory
  // holds the return addresses below the top and is brought up to date when we leave
  int pc_r = a.halt, psp_r = 0;
  if (chain >= 0) {
    psp_r = *pc_sp;
    pc_r = ln.pcs[(psp_r - 1) * L + lane];
  }
#endif

  for (;;) {
    if (chain == -1) {
      const unsigned long long c = atomicAdd(a.next_chain, 1ull);
      if ((long long)c < a.z) {
        chain = (long long)c;
        init_lane(a, ln, chain);
#ifdef LSB_GENERATED
        psp_r = 2;  // init_lane seeded the pc stack [halt, entry]
        pc_r = a.entry;
#endif
      } else {
        chain = -2;
      }
      *my_chain = chain;
    }
#ifdef LSB_GENERATED
    const int pc = chain >= 0 ? pc_r : a.halt;
    const int depth_now = psp_r;
#else
    const int pc = chain >= 0 ? ln.pcs[(*pc_sp - 1) * L + lane] : a.halt;
    const int depth_now = chain >= 0 ? *pc_sp : 0;
#endif
    int b;
    unsigned key = 0, best = 0;
    if (a.sched == LS_SCHED_MOST_POPULATED) {
      const unsigned peers = __match_any_sync(kFull, pc);
      const unsigned k2 = pc == a.halt ? 0u : ((unsigned)__popc(peers) << 16) | (0xffffu - (unsigned)pc);
      const unsigned bm = __reduce_max_sync(kFull, k2);
      b = bm == 0 ? a.halt : (int)(0xffffu - (bm & 0xffffu));
    } else {
      // keyed rules (min_pc, priority, local): the populated block with the least key;
      // keys carry the block index in their low 16 bits (host: schedule.block_keys)
      key = pc == a.halt ? 0xffffffffu : lane_key(a, pc, depth_now);
      best = __reduce_min_sync(kFull, key);
      b = best == 0xffffffffu ? a.halt : (int)(best & 0xffffu);
    }
    if (b == a.halt) {
      if (lane == 0) a.group_done[g] = 1;
      break;
    }
    // another group's fault stops this one within 16 steps (one flag read per 16 steps)
    if ((steps & 15) == 0 && *(volatile int*)a.abort_flag) break;
    if (a.max_steps >= 0 && steps >= a.max_steps) {
      if (lane == 0) a.paused[0] = 1;
      break;
    }
    // specialised builds run a block and its partner (identical code on other variables,
    // codegen.find_pairs) in one step, each lane on its own block
#ifdef LSB_GENERATED
    const int pb = a.sched == LS_SCHED_LOCAL ? -1 : lsbgen::gen_pair(b);
#else
    const int pb = -1;
#endif
    const bool active = (a.sched == LS_SCHED_MOST_POPULATED ? pc == b : (pc != a.halt && key == best)) ||
                        (pb >= 0 && pc == pb);
    const int count = __popc(__ballot_sync(kFull, active));
    const int count_pb = pb >= 0 ? __popc(__ballot_sync(kFull, active && pc == pb)) : 0;
    if (active && a.lane_trace != nullptr) lane_trace_put(a, chain, pc);
    StepFault f;
#if LSB_BLOCK_PROFILE
    const long long t_start = clock64();
#endif
#ifdef LSB_GENERATED
    const bool halted_now = lsbgen::gen_exec_block(a, ln, b, active, chain, f, my_smem, pc_r, psp_r);
#else
    const bool halted_now = LSB_WARP_EXEC(a, ln, b, active, chain, f, my_smem);
#endif
    // per-block statistics as fire-and-forget reductions (no read-modify-write stall)
#if LSB_BLOCK_PROFILE
    if (lane == 0) atomicAdd((unsigned long long*)&bcycles[b], (unsigned long long)(clock64() - t_start));
#endif
    const unsigned fkey = f.pos ? ((unsigned)(f.pos - 1) << 5) | (unsigned)lane : ~0u;
    const unsigned wmin = __reduce_min_sync(kFull, fkey);
    if (wmin != ~0u) {
      if (fkey == wmin) {
        // several groups may fault in one launch: each writes its own slot (no race) and
        // the host reports the lowest chain
        FaultRec& fr = a.fault[g];
        fr.key = (unsigned long long)chain;
        fr.kind = f.kind;
        fr.var = f.var;
        fr.block = pc;  // the lane's own block (b or its partner)
        fr.detail = f.detail;
        fr.chain = chain;
        __threadfence();
        atomicExch(a.abort_flag, 1);
      }
      ++steps;
      break;
    }
    const unsigned hmask = __ballot_sync(kFull, halted_now);
    if (hmask) {
      warp_write_outputs(a, ln, hmask, chain);
      if (halted_now) {
        chain = -1;
        *my_chain = -1;
      }
    }
    if (lane == 0) {
      const int grads = __ldg(&a.blocks[b].grads);
      const int count_b = count - count_pb;
      if (a.gtrace != nullptr) {  // the group's schedule trace (reference ScheduleTrace.record)
        int n = a.gtrace_len[g];
        int* rec = a.gtrace + (size_t)g * a.gtrace_cap;
        if (count_b && n < a.gtrace_cap) rec[n] = b | (count_b << 16);
        n += count_b ? 1 : 0;
        if (count_pb && n < a.gtrace_cap) rec[n] = pb | (count_pb << 16);
        a.gtrace_len[g] = n + (count_pb ? 1 : 0);
      }
      atomicAdd((unsigned long long*)&bsteps[b], 1ull);
      atomicAdd((unsigned long long*)&bactive[b], (unsigned long long)count_b);
      useful += (unsigned long long)count_b * (unsigned long long)grads;
      launched += (unsigned long long)L * (unsigned long long)grads;
      if (count_pb) {
        const int grads_pb = __ldg(&a.blocks[pb].grads);
        atomicAdd((unsigned long long*)&bsteps[pb], 1ull);
        atomicAdd((unsigned long long*)&bactive[pb], (unsigned long long)count_pb);
        useful += (unsigned long long)count_pb * (unsigned long long)grads_pb;
        launched += (unsigned long long)L * (unsigned long long)grads_pb;
      }
    }
    ++steps;
  }
#ifdef LSB_GENERATED
  if (chain >= 0) {  // paused, aborted or faulted with a live chain: pc state back to memory
    ln.pcs[(psp_r - 1 < 0 ? 0 : psp_r - 1) * L + lane] = pc_r;
    *pc_sp = psp_r;
  }
#endif
  if (lane == 0) {
    a.group_steps[g] = steps;
    if (useful) atomicAdd(a.useful, useful);
    if (launched) atomicAdd(a.launched, launched);
  }
}

__global__ void __launch_bounds__(32 * kWarpCtaMax, 1) vm_warp_kernel(const __grid_constant__ VMArgs a) {
  extern __shared__ double lf_smem[];
  // stage the target's B fragments once per CTA; every warp's DMMA reads them at LDS latency
  if (a.stage_doubles > 0) {
    const double2* src = reinterpret_cast<const double2*>(a.stage_src);
    double2* dst = reinterpret_cast<double2*>(lf_smem);
    for (int i = threadIdx.x; i < a.stage_doubles / 2; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
  }
  if (a.tc_img != nullptr) tc_cta_begin(a, reinterpret_cast<unsigned char*>(lf_smem));
  const int g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g < a.n_groups && !a.group_done[g]) warp_group_run(a, lf_smem);
  if (a.wg) wg_leave();  // peers stop waiting for this warp at their superblocks
  if (a.tc_img != nullptr) tc_cta_end();
}

__global__ void init_static_kernel(const __grid_constant__ VMArgs a) {
  const int t = threadIdx.x;
  const long long c = a.chain_of[t];
  if (c < 0) return;
  const Lane ln{a.ws, a.sp, a.pcs, t, a.lanes};
  init_lane(a, ln, c);
}

__global__ void rng_kernel(const int64_t* key, const int64_t* ctr, long long n, double* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = lsb::rng_uniform(key[i], ctr[i]);
}

__global__ void target_eval_kernel(DevTarget tg, int which, const double* x, long long z, double* out,
                                   uint64_t* scratch) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= z) return;
  const int d = tg.dim;
  uint64_t* xs = scratch + i;  // lane-minor copy, stride z
  for (int j = 0; j < d; ++j) xs[(size_t)j * z] = f64_bits(x[(size_t)i * d + j]);
  if (which == 0) {
    out[i] = target_logpdf(tg, xs, (int)z, 1);
  } else {
    uint64_t* gs = scratch + (size_t)d * z + i;
    target_grad(tg, xs, (int)z, gs);
    for (int j = 0; j < d; ++j) out[(size_t)i * d + j] = as_f64(gs[(size_t)j * z]);
  }
}

}  // namespace

// =====================================================================================
// Host side: C ABI
// =====================================================================================

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                                    \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess) return fail(LS_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
static int dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) return fail(LS_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return LS_OK;
}

template <class T>
static int upload(T** d, const std::vector<T>& h) {
  int rc = dalloc(d, h.size());
  if (rc) return rc;
  if (!h.empty()) CK(cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return LS_OK;
}

struct ls_program {
  int device = 0;
  std::vector<ls_block> blocks;
  std::vector<ls_op> ops;
  std::vector<ls_var> vars;
  std::vector<int> inputs;
  int entry = 0, output = 0;
  int n_stacked = 0;
  int flat_rows = 0;
  DevTarget targets[kMaxTargets];
  std::vector<double> host_params[kMaxTargets];  // row-major P (gaussian) for the fp32 image
  std::vector<double*> owned;
};

struct ls_machine {
  ls_program* p = nullptr;
  int device = 0;
  long long z = 0;
  int depth = 0, lanes = 0, groups = 0, group_rows = 0;
  ls_machine_opts opts{};
  std::vector<int> var_row, var_depth, input_width, input_rows;
  RBlock* d_blocks = nullptr;
  ROp* d_ops = nullptr;
  int* d_input_width = nullptr;
  int* d_input_rows = nullptr;
  uint64_t* ws = nullptr;
  int* sp = nullptr;
  int* pcs = nullptr;
  long long* chain_of = nullptr;
  std::vector<uint64_t*> inputs;
  uint64_t** d_input_ptrs = nullptr;
  uint64_t* output = nullptr;
  void* out_host = nullptr;       // ls_machine_set_output_host: page-locked destination
  uint64_t* out_host_dev = nullptr;  // ... and its device alias (written by the kernel)
  int out_width = 0;
  unsigned long long* counters = nullptr;  // [0] next_chain [1] useful [2] launched
  long long* group_steps = nullptr;
  int* group_done = nullptr;
  int* trace_block = nullptr;
  int* trace_active = nullptr;
  long long trace_cap = 0;
  long long* trace_n = nullptr;
  long long* blk_steps = nullptr;
  long long* blk_active = nullptr;
  long long* blk_cycles = nullptr;
  FaultRec* fault = nullptr;
  unsigned* bkey = nullptr;  // [n_blocks] schedule keys
  int* flags = nullptr;  // [0] abort [1] paused-steps [2] paused-trace
  int* lane_trace = nullptr;
  int* lane_trace_len = nullptr;
  int lane_trace_cap = 0;
  int* gtrace = nullptr;
  int* gtrace_len = nullptr;
  int gtrace_cap = 0;
  bool started = false;
  bool warp = false;
  bool refill = false;
  int lf_smem_per_warp = 0;
  int warps_per_cta = 4;     // warp engine CTA shape
  size_t smem_bytes = 0;     // warp engine dynamic shared memory per CTA
  int carveout = -1;         // its preferred shared-memory carveout (cudaSharedmemCarveout*)
  int stage_target = -1;     // target whose B fragments each CTA stages in shared memory
  int stage_doubles = 0;
  // fp32 arm (LS_MF_FP32): tensor-core superblocks, warpgroup stepping
  bool fp32 = false;
  void* tc_img = nullptr;
  int tc_img_bytes = 0, tc_half_bytes = 0, tc_lbo = 0, tc_sbo = 0, tc_smem_off = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  long long launches = 0;
};

static int static_init(ls_machine* m);

// Resolve program ops/blocks against this machine's storage layout (lsb_vm.cuh ROp).
static void resolve(const ls_machine* m, std::vector<ROp>& rops, std::vector<RBlock>& rblocks) {
  const ls_program* p = m->p;
  auto row_of = [&](int v) { return m->var_row[v]; };
  auto sp_of = [&](int v) { return p->vars[v].cls == LS_STACKED ? p->vars[v].sp : -1; };
  rops.resize(p->ops.size());
  for (size_t i = 0; i < p->ops.size(); ++i) {
    const ls_op& o = p->ops[i];
    ROp r{};
    r.opcode = o.opcode; r.action = o.action; r.nin = o.nin; r.kind = o.kind;
    r.width = o.width; r.out = o.out; r.out_row = row_of(o.out); r.out_sp = sp_of(o.out);
    for (int j = 0; j < 3; ++j) {
      if (j < o.nin) {
        const int v = o.in[j];
        r.in_row[j] = row_of(v); r.in_sp[j] = sp_of(v); r.in_w[j] = p->vars[v].width; r.in_kind[j] = p->vars[v].kind;
      } else {
        r.in_row[j] = 0; r.in_sp[j] = -1; r.in_w[j] = 1; r.in_kind[j] = 0;
      }
    }
    r.imm0 = o.imm0; r.imm1 = o.imm1; r.imm2 = o.imm2; r.bits = o.bits;
    r.pad = -1;
    // fused leaf logpdf: the superblock writes var (kind >> 1) - 1, the logpdf op
    // reads var bits - 1 (lowering.fuse_leaf_logpdf); -1 = none
    if (o.opcode == LS_OP_LEAPFROG && (o.kind >> 1) > 0) r.pad = row_of((o.kind >> 1) - 1);
    if (o.opcode == LS_OP_LOGPDF && o.bits > 0) r.pad = row_of((int)o.bits - 1);
    if (o.opcode == LS_OP_LEAPFROG) {  // side outputs as rows (g may be dead: -1)
      const int gv = (int)(o.bits & 0xffffffff), iv = (int)(o.bits >> 32);
      const long long grow = gv >= 0 ? row_of(gv) : -1;
      const long long irow = iv >= 0 ? row_of(iv) : -1;
      r.bits = (long long)((unsigned long long)(grow & 0xffffffff) | ((unsigned long long)irow << 32));
    }
    rops[i] = r;
  }
  rblocks.resize(p->blocks.size());
  for (size_t b = 0; b < p->blocks.size(); ++b) {
    const ls_block& o = p->blocks[b];
    RBlock r{};
    r.op_begin = o.op_begin; r.op_count = o.op_count; r.term = o.term; r.a = o.a; r.b = o.b;
    r.grads = o.grads;
    if (o.term == LS_BRANCH) {
      r.cond_row = row_of(o.cond); r.cond_sp = sp_of(o.cond); r.cond_w = p->vars[o.cond].width;
    } else {
      r.cond_row = 0; r.cond_sp = -1; r.cond_w = 1;
    }
    rblocks[b] = r;
  }
}

static VMArgs make_args(ls_machine* m, long long max_steps) {
  ls_program* p = m->p;
  VMArgs a{};
  a.blocks = m->d_blocks; a.ops = m->d_ops;
  a.n_blocks = (int)p->blocks.size(); a.halt = (int)p->blocks.size(); a.entry = p->entry;
  a.n_inputs = (int)p->inputs.size(); a.input_rows = m->d_input_rows;
  a.output_row = m->var_row[p->output];
  a.output_sp = p->vars[p->output].cls == LS_STACKED ? p->vars[p->output].sp : -1;
  a.out_width = m->out_width;
  a.n_sp_rows = p->n_stacked + 1;
  for (int i = 0; i < kMaxTargets; ++i) a.targets[i] = p->targets[i];
  a.z = m->z; a.depth = m->depth; a.lanes = m->lanes; a.group_rows = m->group_rows;
  a.ws = m->ws; a.sp = m->sp; a.pcs = m->pcs; a.chain_of = m->chain_of;
  a.inputs = (const uint64_t* const*)m->d_input_ptrs; a.input_width = m->d_input_width;
  a.output = m->out_host_dev ? m->out_host_dev : m->output;
  a.next_chain = m->counters + 0;
  a.refill = m->refill;
  a.sched = m->opts.sched;
  a.exact_logpdf = m->opts.exact_logpdf;
  a.max_steps = max_steps;
  a.group_steps = m->group_steps; a.group_done = m->group_done;
  a.trace_block = m->trace_block; a.trace_active = m->trace_active;
  a.trace_cap = m->trace_cap; a.trace_n = m->trace_n;
  a.blk_steps = m->blk_steps; a.blk_active = m->blk_active; a.blk_cycles = m->blk_cycles;
  a.useful = m->counters + 1; a.launched = m->counters + 2;
  a.n_groups = m->groups;
  a.lf_smem_per_warp = m->lf_smem_per_warp;
  a.stage_target = m->stage_target;
  a.stage_doubles = m->stage_doubles;
  a.stage_src = m->stage_target >= 0 ? p->targets[m->stage_target].B1 : nullptr;
  a.lane_trace = m->lane_trace; a.lane_trace_len = m->lane_trace_len; a.lane_trace_cap = m->lane_trace_cap;
  a.gtrace = m->gtrace; a.gtrace_len = m->gtrace_len; a.gtrace_cap = m->gtrace_cap;
  a.fault = m->fault; a.abort_flag = m->flags + 0; a.paused = m->flags + 1;
  a.bkey = m->bkey;
  a.wg = m->fp32 ? 1 : 0;
  a.tc_img = m->tc_img;
  a.tc_img_bytes = m->tc_img_bytes; a.tc_half_bytes = m->tc_half_bytes;
  a.tc_lbo = m->tc_lbo; a.tc_sbo = m->tc_sbo; a.tc_smem_off = m->tc_smem_off;
  return a;
}

extern "C" {

int ls_abi_version(void) { return LS_ABI_VERSION; }

const char* ls_last_error(void) { return g_err.c_str(); }

int ls_device_count(int32_t* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *n = 0;
    cudaGetLastError();
    return fail(LS_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  *n = c;
  return LS_OK;
}

int ls_set_device(int32_t device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    cudaGetLastError();
    return fail(LS_ECUDA, "ls_set_device: no such CUDA device");
  }
  CK(cudaSetDevice(device));
  return LS_OK;
}

int ls_machine_info(const ls_machine* m, int32_t* device, int32_t* groups, int32_t* lanes_per_group) {
  if (!m) return fail(LS_EINVAL, "null machine");
  if (device) *device = m->device;
  if (groups) *groups = m->groups;
  if (lanes_per_group) *lanes_per_group = m->lanes;
  return LS_OK;
}

int ls_program_create(const ls_program_desc* d, ls_program** out) {
  if (!d || !out || d->n_blocks < 1 || d->n_vars < 1) return fail(LS_EINVAL, "empty program");
  auto* p = new ls_program();
  cudaGetDevice(&p->device);
  cudaGetLastError();
  p->blocks.assign(d->blocks, d->blocks + d->n_blocks);
  p->ops.assign(d->ops, d->ops + d->n_ops);
  p->vars.assign(d->vars, d->vars + d->n_vars);
  p->inputs.assign(d->inputs, d->inputs + d->n_inputs);
  p->entry = d->entry;
  p->output = d->output;
  p->flat_rows = d->flat_rows;
  for (auto& v : p->vars)
    if (v.cls == LS_STACKED) p->n_stacked = std::max(p->n_stacked, v.sp + 1);
  for (auto& b : p->blocks) {
    if (b.op_begin < 0 || b.op_begin + b.op_count > d->n_ops) {
      delete p;
      return fail(LS_EINVAL, "block op range");
    }
  }
  *out = p;
  return LS_OK;
}

int ls_program_bind_target(ls_program* p, int32_t slot, int32_t kind, int32_t dim, int32_t n,
                           const double* params, double norm) {
  if (!p || slot < 0 || slot >= kMaxTargets || dim < 1) return fail(LS_EINVAL, "bad target slot");
  CK(cudaSetDevice(p->device));
  const int rows = kind == LS_TARGET_GAUSSIAN ? dim : n;
  if (rows < 1) return fail(LS_EINVAL, "bad target shape");
  std::vector<double> h(params, params + (size_t)rows * dim), ht((size_t)rows * dim);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < dim; ++j) ht[(size_t)j * rows + i] = h[(size_t)i * dim + j];
  double *dP = nullptr, *dPT = nullptr;
  int rc;
  if ((rc = upload(&dP, h)) || (rc = upload(&dPT, ht))) return rc;
  p->owned.push_back(dP);
  p->owned.push_back(dPT);
  DevTarget t{};
  t.kind = kind; t.dim = dim; t.n = n; t.P = dP; t.PT = dPT; t.norm = norm;
  // B operand(s) in DMMA fragment order: Bf[(ks*NT + nt)*32 + l] = B[4ks + l%4][8nt + l/4]
  auto frag = [&](int K, int N, auto at, const double** dst, int* KS, int* NT) -> int {
    *KS = (K + 3) / 4;
    *NT = (N + 7) / 8;
    std::vector<double> f((size_t)(*KS) * (*NT) * 32, 0.0);
    for (int ks = 0; ks < *KS; ++ks)
      for (int nt = 0; nt < *NT; ++nt)
        for (int l = 0; l < 32; ++l) {
          const int k = 4 * ks + l % 4, c = 8 * nt + l / 4;
          if (k < K && c < N) f[((size_t)ks * (*NT) + nt) * 32 + l] = at(k, c);
        }
    double* df = nullptr;
    int rc2 = upload(&df, f);
    if (rc2) return rc2;
    p->owned.push_back(df);
    *dst = df;
    return LS_OK;
  };
  if (kind == LS_TARGET_GAUSSIAN) {
    if ((rc = frag(dim, dim, [&](int k, int c) { return h[(size_t)k * dim + c]; }, &t.B1, &t.KS1, &t.NT1))) return rc;
  } else {
    if ((rc = frag(dim, n, [&](int k, int c) { return h[(size_t)c * dim + k]; }, &t.B1, &t.KS1, &t.NT1))) return rc;
    if ((rc = frag(n, dim, [&](int k, int c) { return h[(size_t)k * dim + c]; }, &t.B2, &t.KS2, &t.NT2))) return rc;
  }
  p->targets[slot] = t;
  p->host_params[slot] = h;
  return LS_OK;
}

int ls_program_destroy(ls_program* p) {
  if (!p) return LS_OK;
  cudaSetDevice(p->device);
  for (double* q : p->owned) cudaFree(q);
  delete p;
  return LS_OK;
}

int ls_machine_destroy(ls_machine* m) {
  if (!m) return LS_OK;
  cudaSetDevice(m->device);
  if (m->stream) cudaStreamSynchronize(m->stream);
  cudaFree(m->d_blocks); cudaFree(m->d_ops); cudaFree(m->d_input_width); cudaFree(m->d_input_rows);
  cudaFree(m->ws); cudaFree(m->sp); cudaFree(m->pcs); cudaFree(m->chain_of);
  for (auto* q : m->inputs) cudaFree(q);
  cudaFree(m->d_input_ptrs); cudaFree(m->output); cudaFree(m->counters);
  cudaFree(m->group_steps); cudaFree(m->group_done); cudaFree(m->trace_block);
  cudaFree(m->trace_active); cudaFree(m->trace_n); cudaFree(m->blk_steps);
  cudaFree(m->blk_active); cudaFree(m->blk_cycles); cudaFree(m->fault); cudaFree(m->flags);
  cudaFree(m->lane_trace); cudaFree(m->lane_trace_len); cudaFree(m->gtrace); cudaFree(m->gtrace_len); cudaFree(m->bkey); cudaFree(m->tc_img);
  if (m->ev0) cudaEventDestroy(m->ev0);
  if (m->ev1) cudaEventDestroy(m->ev1);
  if (m->stream) cudaStreamDestroy(m->stream);
  delete m;
  return LS_OK;
}

static int reset_state(ls_machine* m) {
  const size_t L = m->lanes, nb = m->p->blocks.size();
  const int n_sp_rows = m->p->n_stacked + 1;
  CK(cudaMemsetAsync(m->sp, 0, (size_t)m->groups * n_sp_rows * L * sizeof(int), m->stream));
  CK(cudaMemsetAsync(m->pcs, 0, (size_t)m->groups * (m->depth + 1) * L * sizeof(int), m->stream));
  CK(cudaMemsetAsync(m->counters, 0, 4 * sizeof(unsigned long long), m->stream));
  CK(cudaMemsetAsync(m->group_steps, 0, m->groups * sizeof(long long), m->stream));
  CK(cudaMemsetAsync(m->group_done, 0, m->groups * sizeof(int), m->stream));
  CK(cudaMemsetAsync(m->blk_steps, 0, (size_t)m->groups * nb * sizeof(long long), m->stream));
  CK(cudaMemsetAsync(m->blk_active, 0, (size_t)m->groups * nb * sizeof(long long), m->stream));
  CK(cudaMemsetAsync(m->blk_cycles, 0, (size_t)m->groups * nb * sizeof(long long), m->stream));
  CK(cudaMemsetAsync(m->flags, 0, 4 * sizeof(int), m->stream));
  CK(cudaMemsetAsync(m->trace_n, 0, sizeof(long long), m->stream));
  if (m->lane_trace_len) CK(cudaMemsetAsync(m->lane_trace_len, 0, (size_t)m->z * sizeof(int), m->stream));
  if (m->gtrace_len) CK(cudaMemsetAsync(m->gtrace_len, 0, (size_t)m->groups * sizeof(int), m->stream));
  {
    const FaultRec f0{~0ull, 0, 0, 0, 0, -1};
    std::vector<FaultRec> fr((size_t)m->groups, f0);
    CK(cudaMemcpyAsync(m->fault, fr.data(), fr.size() * sizeof(FaultRec), cudaMemcpyHostToDevice, m->stream));
    CK(cudaStreamSynchronize(m->stream));
  }
  std::vector<long long> slots((size_t)m->groups * L, -1);
  if (!m->refill)
    for (size_t t = 0; t < L; ++t) slots[t] = (long long)t < m->z ? (long long)t : -2;
  CK(cudaMemcpyAsync(m->chain_of, slots.data(), slots.size() * sizeof(long long), cudaMemcpyHostToDevice,
                     m->stream));
  CK(cudaStreamSynchronize(m->stream));
  m->started = false;
  return static_init(m);
}

int ls_machine_create(ls_program* p, int64_t z, int32_t depth, const ls_machine_opts* opts,
                      ls_machine** out) {
  if (!p || !out || z < 1 || depth < 1) return fail(LS_EINVAL, "bad machine arguments");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(LS_ECUDA, "no CUDA device: the lockstep B200 engine has no CPU fallback");
  }
  CK(cudaSetDevice(p->device));  // a machine lives on its program's device
  auto* m = new ls_machine();
  m->p = p;
  m->device = p->device;
  m->z = z;
  m->depth = depth;
  if (opts) m->opts = *opts;
  int dev = p->device, sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int groups;
  m->warp = m->opts.warp_groups != 0;
#ifdef LSB_GENERATED
  if (!m->warp) {
    delete m;
    return fail(LS_EINVAL, "a program-specialised library runs the warp engine only");
  }
#endif
  if (m->warp) {
    // one 32-lane group per warp, 4 warps per CTA; default: a group per 32 chains,
    // capped at the warps that are resident at once (persistent CTAs refill chains)
    m->lanes = 32;
    m->refill = true;
    for (const auto& op : p->ops) {
      if (op.opcode == LS_OP_LEAPFROG)
        m->lf_smem_per_warp = std::max(m->lf_smem_per_warp, lf_smem_doubles(p->targets[op.imm0].dim));
      // DMMA gradients / fast logpdfs stage their A operand as one 8-chain tile
      if ((op.opcode == LS_OP_GRAD || op.opcode == LS_OP_LOGPDF) &&
          p->targets[op.imm0].kind == LS_TARGET_GAUSSIAN && p->targets[op.imm0].NT1 <= kLfRegMaxTiles)
        m->lf_smem_per_warp = std::max(m->lf_smem_per_warp, 8 * lf_stride_q(p->targets[op.imm0].dim));
      // DMMA logistic-regression gradients stage w the same way
      if ((op.opcode == LS_OP_GRAD || op.opcode == LS_OP_LOGPDF) && p->targets[op.imm0].kind == LS_TARGET_LOGREG &&
          p->targets[op.imm0].NT2 <= 16)
        m->lf_smem_per_warp = std::max(m->lf_smem_per_warp, p->targets[op.imm0].n >= kLrStreamMinN
                                                                ? lr_stream_doubles(p->targets[op.imm0].dim)
                                                                : 8 * lf_stride_q(p->targets[op.imm0].dim));
    }
    m->lf_smem_per_warp = (m->lf_smem_per_warp + 1) & ~1;  // 16-byte aligned per-warp areas
#if defined(LSB_GENERATED) && LSB_GEN_STAGED
    // generated block code stages long copies through 48 rows x 32 lanes per warp
    m->lf_smem_per_warp = std::max(m->lf_smem_per_warp, 48 * 32);
#endif
    const long long want = (z + 31) / 32;
    // Stage one gaussian target's B fragments per CTA when every superblock uses it:
    // CTAs of up to 16 warps (one per SM) share the copy. Otherwise 4-warp CTAs.
    int st = -1;
    bool one = true;
    for (const auto& op : p->ops)
      if (op.opcode == LS_OP_LEAPFROG) {
        if (st >= 0 && st != op.imm0) one = false;
        st = op.imm0;
      }
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (st >= 0 && one && !(m->opts.flags & LS_MF_NO_STAGE) && p->targets[st].kind == LS_TARGET_GAUSSIAN) {
      const int sd = p->targets[st].KS1 * p->targets[st].NT1 * 32;
      // enough warps per CTA that one CTA per SM covers the groups, 4..16
      int wpc = (int)std::min<long long>(kWarpCtaMax, std::max<long long>(4, (want + sms - 1) / sms));
      while (wpc >= 4 && ((size_t)sd + (size_t)wpc * m->lf_smem_per_warp) * sizeof(double) > (size_t)smem_optin) --wpc;
      if (wpc >= 4) {
        m->stage_target = st;
        m->stage_doubles = sd;
        m->warps_per_cta = wpc;
      }
    }
    if (m->opts.flags & LS_MF_FP32) {
      // fp32 arm: the superblock target's precision matrix as a TF32 hi/lo image (UMMA K-major,
      // no swizzle) that each CTA bulk-copies into shared memory in place of the DMMA fragments
      if (st < 0 || !one || p->targets[st].kind != LS_TARGET_GAUSSIAN || p->targets[st].dim > 128) {
        delete m;
        return fail(LS_EINVAL, "the fp32 arm needs fused leapfrogs of one gaussian target with d <= 128");
      }
      m->fp32 = true;
      m->stage_target = -1;
      m->stage_doubles = 0;
      // the tensor-core superblock needs no per-warp shared tiles; other DMMA contractions
      // (the iteration's initial logpdf) read their A operand from the workspace (measured
      // faster than staging it: the freed shared memory goes to L1)
      m->lf_smem_per_warp = 0;
      const int d = p->targets[st].dim, K = (d + 7) / 8 * 8, N = (d + 15) / 16 * 16;
      std::vector<float> P32((size_t)K * N, 0.f);
      const std::vector<double>& hp = p->host_params[st];
      for (int k = 0; k < d; ++k)
        for (int n = 0; n < d; ++n) P32[(size_t)k * N + n] = (float)hp[(size_t)k * d + n];
      std::vector<uint8_t> img;
      m->tc_lbo = 128;
      m->tc_sbo = (K / 4) * 128;
      m->tc_half_bytes = lsbtc::b_image_nosw(P32.data(), K, N, N, m->tc_lbo, m->tc_sbo, img);
      m->tc_img_bytes = (int)img.size();
      int rc2 = dalloc((uint8_t**)&m->tc_img, img.size());
      if (rc2) {
        delete m;
        return rc2;
      }
      CK(cudaMemcpy(m->tc_img, img.data(), img.size(), cudaMemcpyHostToDevice));
      // one CTA per SM (it owns the SM's tensor memory), enough warps to cover the groups
      int wpc = (int)std::min<long long>(kWarpCtaMax, std::max<long long>(4, (want + sms - 1) / sms));
      auto off_of = [&](int w) { return ((size_t)w * m->lf_smem_per_warp * sizeof(double) + 1023) / 1024 * 1024; };
      while (wpc >= 1 && off_of(wpc) + img.size() > (size_t)smem_optin) --wpc;
      if (wpc < 1) {
        cudaFree(m->tc_img);
        delete m;
        return fail(LS_EINVAL, "the fp32 arm's shared-memory image does not fit");
      }
      m->warps_per_cta = wpc;
      m->tc_smem_off = (int)off_of(wpc);
    }
    if (!m->fp32 && m->stage_target < 0)  // large per-warp scratch (streamed designs): smaller CTAs
      while (m->warps_per_cta > 1 && (size_t)m->warps_per_cta * m->lf_smem_per_warp * sizeof(double) > (size_t)smem_optin)
        --m->warps_per_cta;
    const size_t smem = m->fp32 ? (size_t)m->tc_smem_off + (size_t)m->tc_img_bytes
                                : ((size_t)m->stage_doubles + (size_t)m->warps_per_cta * m->lf_smem_per_warp) * sizeof(double);
    m->smem_bytes = smem;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(vm_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // machines with large per-warp scratch (not the staged-target or fp32 CTAs, which hold
    // one CTA per SM by design) let the whole unified L1/shared array go to shared
    // memory: without that preference the occupancy query (and the launch) size the
    // carveout for one such CTA per SM (measured: 1 CTA of 62.6 KB where 3 fit); the others
    // keep the default split (L1 for the block code's loads). Set again at every launch.
    m->carveout = (smem > 48 * 1024 && !m->fp32 && m->stage_target < 0) ? (int)cudaSharedmemCarveoutMaxShared
                                                                          : (int)cudaSharedmemCarveoutDefault;
    cudaFuncSetAttribute(vm_warp_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, m->carveout);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vm_warp_kernel, 32 * m->warps_per_cta, smem) !=
            cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    groups = m->opts.ctas > 0 ? 4 * m->opts.ctas
                              : (int)std::min<long long>(want, (long long)sms * m->warps_per_cta * per_sm);
    if (groups > want) groups = (int)want;
    if (m->fp32 && m->opts.ctas > 0) groups = m->warps_per_cta * m->opts.ctas;
  } else {
    int lanes = m->opts.lanes_per_cta > 0 ? m->opts.lanes_per_cta : (int)std::min<long long>(z, kMaxLanes);
    if (m->opts.lanes_per_cta <= 0 && z > kMaxLanes) {
      delete m;
      return fail(LS_EINVAL, "a single schedule group holds at most 1024 lanes; set lanes_per_cta");
    }
    lanes = std::min(kMaxLanes, ((lanes + 31) / 32) * 32);
    m->lanes = lanes;
    m->refill = z > lanes;
    const long long want = (z + lanes - 1) / lanes;
    groups = m->opts.ctas > 0 ? m->opts.ctas : sms * std::max(1, 1024 / lanes);
    if (!m->refill) groups = 1;
    if (groups > want) groups = (int)want;
  }
  m->groups = groups;
  if (m->opts.trace && groups != 1) {
    delete m;
    return fail(LS_EINVAL, "per-step traces need a single schedule group (z <= lanes_per_cta)");
  }
  // storage layout: the lowering placed every non-stacked variable in the flat
  // region; stacked variables follow with depth slots each
  const auto& vars = p->vars;
  m->var_row.resize(vars.size());
  m->var_depth.resize(vars.size());
  int rows = p->flat_rows;
  for (size_t v = 0; v < vars.size(); ++v) {
    const int slots = vars[v].cls == LS_STACKED ? depth : 1;
    m->var_depth[v] = slots;
    if (vars[v].cls == LS_STACKED) {
      m->var_row[v] = rows;
      rows += slots * vars[v].width;
    } else {
      m->var_row[v] = vars[v].row;
      if (vars[v].row < 0 || vars[v].row + vars[v].width > p->flat_rows) {
        delete m;
        return fail(LS_EINVAL, "variable rows outside the flat region");
      }
    }
  }
  m->group_rows = rows;
  m->out_width = vars[p->output].width;
  for (int v : p->inputs) {
    m->input_width.push_back(vars[v].width);
    m->input_rows.push_back(m->var_row[v]);
  }
  const int n_sp_rows = p->n_stacked + 1;
  const size_t L = m->lanes;
  std::vector<ROp> rops;
  std::vector<RBlock> rblocks;
  resolve(m, rops, rblocks);
  int rc = 0;
  CK(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
  if ((rc = upload(&m->d_ops, rops)) || (rc = upload(&m->d_blocks, rblocks)) ||
      (rc = upload(&m->d_input_width, m->input_width)) || (rc = upload(&m->d_input_rows, m->input_rows)) ||
      (rc = dalloc(&m->ws, (size_t)groups * rows * L)) ||
      (rc = dalloc(&m->sp, (size_t)groups * n_sp_rows * L)) ||
      (rc = dalloc(&m->pcs, (size_t)groups * (depth + 1) * L)) ||
      (rc = dalloc(&m->chain_of, (size_t)groups * L)) ||
      (rc = dalloc(&m->d_input_ptrs, std::max<size_t>(1, p->inputs.size()))) ||
      (rc = dalloc(&m->output, (size_t)z * m->out_width)) ||
      (rc = dalloc(&m->counters, 4)) || (rc = dalloc(&m->group_steps, groups)) ||
      (rc = dalloc(&m->group_done, groups)) ||
      (rc = dalloc(&m->blk_steps, (size_t)groups * p->blocks.size())) ||
      (rc = dalloc(&m->blk_active, (size_t)groups * p->blocks.size())) ||
      (rc = dalloc(&m->blk_cycles, (size_t)groups * p->blocks.size())) ||
      (rc = dalloc(&m->fault, (size_t)groups)) || (rc = dalloc(&m->flags, 4)) || (rc = dalloc(&m->trace_n, 1))) {
    ls_machine_destroy(m);
    return rc;
  }
  {
    std::vector<unsigned> keys(p->blocks.size());
    for (size_t b = 0; b < keys.size(); ++b) keys[b] = (unsigned)b;  // reference min-pc
    if ((rc = upload(&m->bkey, keys))) {
      ls_machine_destroy(m);
      return rc;
    }
  }
  for (size_t k = 0; k < p->inputs.size(); ++k) {
    uint64_t* buf = nullptr;
    if ((rc = dalloc(&buf, (size_t)z * m->input_width[k]))) {
      ls_machine_destroy(m);
      return rc;
    }
    cudaMemsetAsync(buf, 0, (size_t)z * m->input_width[k] * 8, m->stream);
    m->inputs.push_back(buf);
  }
  if (!m->inputs.empty())
    CK(cudaMemcpy(m->d_input_ptrs, m->inputs.data(), m->inputs.size() * sizeof(uint64_t*), cudaMemcpyHostToDevice));
  // the reference zero-fills all storage at init (pc_vm.py:171-181)
  CK(cudaMemsetAsync(m->ws, 0, (size_t)groups * rows * L * sizeof(uint64_t), m->stream));
  CK(cudaMemsetAsync(m->output, 0, (size_t)z * m->out_width * sizeof(uint64_t), m->stream));
  if (m->opts.lane_trace_cap > 0) {
    m->lane_trace_cap = m->opts.lane_trace_cap;
    if ((rc = dalloc(&m->lane_trace, (size_t)z * m->lane_trace_cap)) || (rc = dalloc(&m->lane_trace_len, (size_t)z))) {
      ls_machine_destroy(m);
      return rc;
    }
  }
  if (m->opts.group_trace_cap > 0) {
    if (!m->warp) {
      ls_machine_destroy(m);
      return fail(LS_EINVAL, "group traces are recorded by the warp engine (warp_groups = 1)");
    }
    m->gtrace_cap = m->opts.group_trace_cap;
    if ((rc = dalloc(&m->gtrace, (size_t)groups * m->gtrace_cap)) || (rc = dalloc(&m->gtrace_len, (size_t)groups))) {
      ls_machine_destroy(m);
      return rc;
    }
  }
  if (m->opts.trace) {
    m->trace_cap = 1 << 16;
    if ((rc = dalloc(&m->trace_block, m->trace_cap)) || (rc = dalloc(&m->trace_active, m->trace_cap))) {
      ls_machine_destroy(m);
      return rc;
    }
  }
  if ((rc = reset_state(m))) {
    ls_machine_destroy(m);
    return rc;
  }
  *out = m;
  return LS_OK;
}

int ls_machine_set_block_keys(ls_machine* m, const uint32_t* keys, int32_t n_blocks) {
  if (!m || !keys || n_blocks != (int32_t)m->p->blocks.size()) return fail(LS_EINVAL, "bad block keys");
  CK(cudaSetDevice(m->device));
  for (int b = 0; b < n_blocks; ++b)
    if ((int)(keys[b] & 0xffffu) != b || keys[b] == 0xffffffffu)
      return fail(LS_EINVAL, "block key must carry its block index in bits 0..15");
  CK(cudaMemcpy(m->bkey, keys, (size_t)n_blocks * sizeof(unsigned), cudaMemcpyHostToDevice));
  return LS_OK;
}

int ls_machine_reset(ls_machine* m) {
  if (!m) return fail(LS_EINVAL, "null machine");
  CK(cudaSetDevice(m->device));
  return reset_state(m);
}

int ls_machine_set_input(ls_machine* m, int32_t idx, const void* host, int64_t bytes) {
  if (!m || idx < 0 || idx >= (int)m->inputs.size()) return fail(LS_EINVAL, "bad input index");
  CK(cudaSetDevice(m->device));
  if (bytes != m->z * m->input_width[idx] * 8) return fail(LS_EINVAL, "input size mismatch");
  CK(cudaMemcpyAsync(m->inputs[idx], host, bytes, cudaMemcpyHostToDevice, m->stream));
  CK(cudaStreamSynchronize(m->stream));
  return static_init(m);
}

int ls_machine_set_input_device(ls_machine* m, int32_t idx, const void* dev, int64_t bytes) {
  if (!m || idx < 0 || idx >= (int)m->inputs.size()) return fail(LS_EINVAL, "bad input index");
  CK(cudaSetDevice(m->device));
  if (bytes != m->z * m->input_width[idx] * 8) return fail(LS_EINVAL, "input size mismatch");
  CK(cudaMemcpyAsync(m->inputs[idx], dev, bytes, cudaMemcpyDeviceToDevice, m->stream));
  return static_init(m);
}

}  // extern "C"

// Single-group machines are seeded eagerly (pc stack [halt, entry], one live
// slot per data stack, inputs in slot 0) so observers can inspect them before
// the first step; refilling machines seed each lane when it takes a chain.
static int static_init(ls_machine* m) {
  if (m->refill || m->started) return LS_OK;
  VMArgs a = make_args(m, 0);
  init_static_kernel<<<1, m->lanes, 0, m->stream>>>(a);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(m->stream));
  return LS_OK;
}

extern "C" {

int ls_run(ls_machine* m, int64_t max_steps, ls_status* st) {
  if (!m || !st) return fail(LS_EINVAL, "null machine");
  CK(cudaSetDevice(m->device));
  ls_program* p = m->p;
  VMArgs a = make_args(m, max_steps);
  m->started = true;
  size_t smem = m->warp ? m->smem_bytes : (p->blocks.size() + 1) * sizeof(int);
  if (smem > 48 * 1024) {
    if (m->warp) CK(cudaFuncSetAttribute(vm_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    else CK(cudaFuncSetAttribute(vm_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  if (m->warp) CK(cudaFuncSetAttribute(vm_warp_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, m->carveout));
  CK(cudaMemsetAsync(m->flags + 1, 0, 2 * sizeof(int), m->stream));
  if (!m->ev0) {
    CK(cudaEventCreate(&m->ev0));
    CK(cudaEventCreate(&m->ev1));
  }
  CK(cudaEventRecord(m->ev0, m->stream));
  if (m->warp)
    vm_warp_kernel<<<(m->groups + m->warps_per_cta - 1) / m->warps_per_cta, 32 * m->warps_per_cta, smem, m->stream>>>(a);
  else vm_cta_kernel<<<m->groups, m->lanes, smem, m->stream>>>(a);
  CK(cudaGetLastError());
  CK(cudaEventRecord(m->ev1, m->stream));
  CK(cudaStreamSynchronize(m->stream));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
  m->launches += 1;
  int flags[3];
  FaultRec f;
  std::vector<long long> gsteps(m->groups);
  std::vector<int> gdone(m->groups);
  unsigned long long cnt[3];
  CK(cudaMemcpy(flags, m->flags, sizeof(flags), cudaMemcpyDeviceToHost));
  {
    std::vector<FaultRec> fr((size_t)m->groups);
    CK(cudaMemcpy(fr.data(), m->fault, fr.size() * sizeof(FaultRec), cudaMemcpyDeviceToHost));
    f = fr[0];
    for (const auto& x : fr)  // the lowest chain among the groups that faulted
      if (x.chain >= 0 && (f.chain < 0 || x.chain < f.chain)) f = x;
  }
  CK(cudaMemcpy(gsteps.data(), m->group_steps, m->groups * sizeof(long long), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(gdone.data(), m->group_done, m->groups * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cnt, m->counters, sizeof(cnt), cudaMemcpyDeviceToHost));
  std::memset(st, 0, sizeof(*st));
  st->steps = *std::max_element(gsteps.begin(), gsteps.end());
  st->useful_grads = (int64_t)cnt[1];
  st->launched_grads = (int64_t)cnt[2];
  st->kernel_ms = ms;
  st->launches = m->launches;
  st->var = -1;
  if (flags[0]) {
    st->kind = f.kind;
    st->var = f.var;
    st->lane = f.chain;
    st->block = f.block;
    st->pad = f.detail;
    return LS_OK;
  }
  bool all_done = true;
  for (int d : gdone) all_done = all_done && d;
  if (all_done) st->kind = LS_RUN_HALTED;
  else if (flags[1] && max_steps >= 0 && st->steps >= max_steps) st->kind = LS_RUN_STEP_LIMIT;
  else st->kind = LS_RUN_PAUSED;
  return LS_OK;
}

int ls_read_output(ls_machine* m, void* host, int64_t bytes) {
  if (!m) return fail(LS_EINVAL, "null machine");
  CK(cudaSetDevice(m->device));
  if (bytes != m->z * m->out_width * 8) return fail(LS_EINVAL, "output size mismatch");
  if (m->out_host_dev) {  // the kernel wrote the rows straight into the host buffer
    CK(cudaStreamSynchronize(m->stream));
    if (host != m->out_host) std::memcpy(host, m->out_host, (size_t)bytes);
    return LS_OK;
  }
  CK(cudaMemcpyAsync(host, m->output, bytes, cudaMemcpyDeviceToHost, m->stream));
  CK(cudaStreamSynchronize(m->stream));
  return LS_OK;
}

int ls_machine_set_output_host(ls_machine* m, void* host, int64_t bytes) {
  if (!m) return fail(LS_EINVAL, "null machine");
  CK(cudaSetDevice(m->device));
  if (!host) {
    m->out_host = nullptr;
    m->out_host_dev = nullptr;
    return LS_OK;
  }
  if (!m->warp) return fail(LS_EINVAL, "host output needs the warp engine");
  if (bytes != m->z * m->out_width * 8) return fail(LS_EINVAL, "output size mismatch");
  void* dev = nullptr;
  if (cudaHostGetDevicePointer(&dev, host, 0) != cudaSuccess) {
    cudaGetLastError();
    return fail(LS_EINVAL, "host output must be mapped page-locked memory (ls_host_alloc)");
  }
  m->out_host = host;
  m->out_host_dev = (uint64_t*)dev;
  return LS_OK;
}

int ls_host_alloc(int64_t bytes, void** host) {
  if (!host || bytes <= 0) return fail(LS_EINVAL, "bad host allocation request");
  *host = nullptr;
  if (cudaHostAlloc(host, (size_t)bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    *host = nullptr;
    return fail(LS_ENOMEM, "cudaHostAlloc failed");
  }
  return LS_OK;
}

int ls_host_free(void* host) {
  if (host) CK(cudaFreeHost(host));
  return LS_OK;
}

int ls_copy_output_device(ls_machine* m, void* dev_dst, int64_t bytes) {
  if (!m || !dev_dst) return fail(LS_EINVAL, "null machine");
  CK(cudaSetDevice(m->device));
  if (bytes <= 0 || bytes > m->z * m->out_width * 8 || bytes % (m->out_width * 8))
    return fail(LS_EINVAL, "output size mismatch (whole rows, at most z of them)");
  CK(cudaMemcpyAsync(dev_dst, m->out_host_dev ? m->out_host_dev : m->output, bytes, cudaMemcpyDefault,
                     m->stream));
  CK(cudaStreamSynchronize(m->stream));
  return LS_OK;
}

int ls_output_device(ls_machine* m, void** dev) {
  if (!m || !dev) return fail(LS_EINVAL, "null machine");
  CK(cudaSetDevice(m->device));
  *dev = m->out_host_dev ? m->out_host_dev : m->output;
  return LS_OK;
}

int ls_trace_fetch(ls_machine* m, int32_t* blocks, int32_t* active, int64_t cap, int64_t* n) {
  if (!m || !n) return fail(LS_EINVAL, "null machine");
  CK(cudaSetDevice(m->device));
  *n = 0;
  if (!m->trace_block) return LS_OK;
  long long have = 0;
  CK(cudaMemcpy(&have, m->trace_n, sizeof(have), cudaMemcpyDeviceToHost));
  const long long k = std::min<long long>(have, cap);
  if (k > 0) {
    CK(cudaMemcpy(blocks, m->trace_block, k * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(active, m->trace_active, k * sizeof(int), cudaMemcpyDeviceToHost));
  }
  if (k < have) {  // keep the undrained tail at the front
    std::vector<int> rb(have - k), ra(have - k);
    CK(cudaMemcpy(rb.data(), m->trace_block + k, (have - k) * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ra.data(), m->trace_active + k, (have - k) * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(m->trace_block, rb.data(), rb.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(m->trace_active, ra.data(), ra.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  const long long rest = have - k;
  CK(cudaMemcpy(m->trace_n, &rest, sizeof(rest), cudaMemcpyHostToDevice));
  *n = k;
  return LS_OK;
}

int ls_block_totals(ls_machine* m, int64_t* steps, int64_t* active) {
  if (!m) return fail(LS_EINVAL, "null machine");
  CK(cudaSetDevice(m->device));
  const size_t nb = m->p->blocks.size();
  std::vector<long long> s((size_t)m->groups * nb), a((size_t)m->groups * nb);
  CK(cudaMemcpy(s.data(), m->blk_steps, s.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(a.data(), m->blk_active, a.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  for (size_t b = 0; b < nb; ++b) {
    long long ss = 0, aa = 0;
    for (int g = 0; g < m->groups; ++g) {
      ss += s[(size_t)g * nb + b];
      aa += a[(size_t)g * nb + b];
    }
    steps[b] = ss;
    active[b] = aa;
  }
  return LS_OK;
}

#if LSB_SB_PROFILE
// dev-only: read and clear the superblock phase clocks (lsb_vm.cuh lsb_sb_prof)
int ls_debug_sb_profile(uint64_t* out8) {
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpyFromSymbol(out8, lsbvm::lsb_sb_prof, 8 * sizeof(uint64_t)));
  static const uint64_t zero[8] = {0};
  CK(cudaMemcpyToSymbol(lsbvm::lsb_sb_prof, zero, sizeof(zero)));
  return LS_OK;
}
#endif

int ls_block_cycles(ls_machine* m, int64_t* cycles) {
  if (!m) return fail(LS_EINVAL, "null machine");
  CK(cudaSetDevice(m->device));
  const size_t nb = m->p->blocks.size();
  std::vector<long long> c((size_t)m->groups * nb);
  CK(cudaMemcpy(c.data(), m->blk_cycles, c.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  for (size_t b = 0; b < nb; ++b) {
    long long cc = 0;
    for (int g = 0; g < m->groups; ++g) cc += c[(size_t)g * nb + b];
    cycles[b] = cc;
  }
  return LS_OK;
}

int ls_read_var(ls_machine* m, int32_t var, void* host, int64_t bytes) {
  if (!m || var < 0 || var >= (int)m->p->vars.size()) return fail(LS_EINVAL, "bad var");
  CK(cudaSetDevice(m->device));
  if (m->groups != 1 || m->refill) return fail(LS_EINVAL, "observer access needs a single schedule group");
  const int slots = m->var_depth[var], w = m->p->vars[var].width;
  const long long z = m->z;
  if (bytes != (int64_t)slots * z * w * 8) return fail(LS_EINVAL, "var size mismatch");
  std::vector<uint64_t> raw((size_t)slots * w * m->lanes);
  CK(cudaMemcpy(raw.data(), m->ws + (size_t)m->var_row[var] * m->lanes, raw.size() * 8, cudaMemcpyDeviceToHost));
  auto* dst = static_cast<uint64_t*>(host);
  for (int s = 0; s < slots; ++s)
    for (long long l = 0; l < z; ++l)
      for (int i = 0; i < w; ++i) dst[((size_t)s * z + l) * w + i] = raw[((size_t)s * w + i) * m->lanes + l];
  return LS_OK;
}

int ls_read_pointers(ls_machine* m, int32_t var, int64_t* host, int64_t z) {
  if (!m || z != m->z) return fail(LS_EINVAL, "bad pointer request");
  CK(cudaSetDevice(m->device));
  if (m->groups != 1 || m->refill) return fail(LS_EINVAL, "observer access needs a single schedule group");
  int row;
  if (var < 0) row = m->p->n_stacked;
  else if (m->p->vars[var].cls == LS_STACKED) row = m->p->vars[var].sp;
  else return fail(LS_EINVAL, "not a stacked variable");
  std::vector<int> raw(m->lanes);
  CK(cudaMemcpy(raw.data(), m->sp + (size_t)row * m->lanes, m->lanes * sizeof(int), cudaMemcpyDeviceToHost));
  for (long long l = 0; l < z; ++l) host[l] = raw[l];
  return LS_OK;
}

int ls_read_pc_stack(ls_machine* m, int32_t* host, int64_t count) {
  if (!m || count != (int64_t)(m->depth + 1) * m->z) return fail(LS_EINVAL, "bad pc request");
  CK(cudaSetDevice(m->device));
  if (m->groups != 1 || m->refill) return fail(LS_EINVAL, "observer access needs a single schedule group");
  std::vector<int> raw((size_t)(m->depth + 1) * m->lanes);
  CK(cudaMemcpy(raw.data(), m->pcs, raw.size() * sizeof(int), cudaMemcpyDeviceToHost));
  for (int s = 0; s <= m->depth; ++s)
    for (long long l = 0; l < m->z; ++l) host[(size_t)s * m->z + l] = raw[(size_t)s * m->lanes + l];
  return LS_OK;
}

int ls_group_trace_fetch(ls_machine* m, int32_t* recs, int32_t* lens, int64_t cap) {
  if (!m || !m->gtrace) return fail(LS_EINVAL, "machine was created without group traces");
  if (cap != m->gtrace_cap) return fail(LS_EINVAL, "group trace capacity mismatch");
  CK(cudaSetDevice(m->device));
  CK(cudaStreamSynchronize(m->stream));
  CK(cudaMemcpy(recs, m->gtrace, (size_t)m->groups * cap * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(lens, m->gtrace_len, (size_t)m->groups * sizeof(int), cudaMemcpyDeviceToHost));
  return LS_OK;
}

int ls_lane_trace_fetch(ls_machine* m, int32_t* blocks, int32_t* lens, int64_t cap) {
  if (!m || !m->lane_trace) return fail(LS_EINVAL, "machine was created without lane traces");
  CK(cudaSetDevice(m->device));
  if (cap != m->lane_trace_cap) return fail(LS_EINVAL, "lane trace capacity mismatch");
  CK(cudaMemcpy(blocks, m->lane_trace, (size_t)m->z * cap * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(lens, m->lane_trace_len, (size_t)m->z * sizeof(int), cudaMemcpyDeviceToHost));
  return LS_OK;
}

int ls_machine_sync(ls_machine* m) {
  if (!m) return fail(LS_EINVAL, "null machine");
  CK(cudaSetDevice(m->device));
  CK(cudaStreamSynchronize(m->stream));
  return LS_OK;
}

int ls_rng_uniform(const int64_t* key, const int64_t* counter, int64_t n, double* out) {
  if (n <= 0) return LS_OK;
  int64_t *dk = nullptr, *dc = nullptr;
  double* dout = nullptr;
  int rc;
  if ((rc = dalloc(&dk, n)) || (rc = dalloc(&dc, n)) || (rc = dalloc(&dout, n))) {
    cudaFree(dk);
    cudaFree(dc);
    return rc;
  }
  cudaMemcpy(dk, key, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, counter, n * 8, cudaMemcpyHostToDevice);
  rng_kernel<<<(unsigned)((n + 255) / 256), 256>>>(dk, dc, n, dout);
  cudaError_t e = cudaMemcpy(out, dout, n * 8, cudaMemcpyDeviceToHost);
  cudaFree(dk);
  cudaFree(dc);
  cudaFree(dout);
  if (e != cudaSuccess) return fail(LS_ECUDA, cudaGetErrorString(e));
  return LS_OK;
}

int ls_target_eval(int32_t kind, int32_t which, int32_t dim, int32_t n, const double* params, double norm,
                   const double* x, int64_t z, double* out) {
  if (z <= 0) return LS_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(LS_ECUDA, "no CUDA device: the lockstep B200 engine has no CPU fallback");
  }
  ls_program tmp;
  int rc = ls_program_bind_target(&tmp, 0, kind, dim, n, params, norm);
  if (rc) {
    for (double* q : tmp.owned) cudaFree(q);
    return rc;
  }
  double *dx = nullptr, *dout = nullptr;
  uint64_t* scratch = nullptr;
  const size_t outn = which == 0 ? (size_t)z : (size_t)z * dim;
  if ((rc = dalloc(&dx, (size_t)z * dim)) || (rc = dalloc(&dout, outn)) ||
      (rc = dalloc(&scratch, (size_t)2 * z * dim))) {
    cudaFree(dx);
    cudaFree(dout);
    for (double* q : tmp.owned) cudaFree(q);
    return rc;
  }
  cudaMemcpy(dx, x, (size_t)z * dim * 8, cudaMemcpyHostToDevice);
  target_eval_kernel<<<(unsigned)((z + 127) / 128), 128>>>(tmp.targets[0], which, dx, z, dout, scratch);
  cudaError_t e = cudaMemcpy(out, dout, outn * 8, cudaMemcpyDeviceToHost);
  cudaFree(dx);
  cudaFree(dout);
  cudaFree(scratch);
  for (double* q : tmp.owned) cudaFree(q);
  if (e != cudaSuccess) return fail(LS_ECUDA, cudaGetErrorString(e));
  return LS_OK;
}

}  // extern "C"
