/*
 * lockstep_b200.h — C ABI of the B200 program-counter VM.
 *
 * This is the drop-in boundary for the reference's execution engine,
 * `lockstep.pc_vm` (reference pkg/src/lockstep/pc_vm.py). Each entry point
 * names the reference interface it replaces:
 *
 *   ls_program_create / ls_program_bind_target
 *       <- the CompiledProgram consumed by pc_vm.init_machine
 *          (compiler.py:52-71, pc_vm.py:140-213) plus the target kernels
 *          registered by workloads._make_target (workloads.py:158-171)
 *   ls_machine_create / ls_machine_set_input
 *       <- pc_vm.init_machine (pc_vm.py:140-213): storage allocation,
 *          data stacks seeded with one live slot, pc stack seeded [halt, entry]
 *   ls_run
 *       <- pc_vm.run_vm / pc_vm.step (pc_vm.py:304-349): batched block steps
 *          until every lane halts, StepLimitExceeded, stack faults
 *   ls_read_output (+ ls_host_alloc / ls_host_free for page-locked destinations)
 *       <- Machine.output_value (pc_vm.py:136-137): a copy of the output var
 *   ls_trace_fetch / ls_block_totals
 *       <- ScheduleTrace.record (metrics.py:36-37), one record per step
 *   ls_read_var / ls_read_pointers
 *       <- Machine.stacks / regs / scratch access by observers (pc_vm.py:323)
 *   ls_rng_uniform
 *       <- runtime.rng_uniform (runtime.py:288-303)
 *   ls_target_eval
 *       <- the logpdf_/grad_ kernels of a TargetDensity (workloads.py:186-228)
 *
 * All functions return LS_OK (0) or a negative LS_E* code; ls_last_error()
 * gives a message. Pointers are plain host pointers unless a name says
 * "device". One machine is confined to one host thread and one CUDA stream.
 * There is no CPU execution path: without a CUDA device every compute entry
 * point fails with LS_ECUDA.
 */
#ifndef LOCKSTEP_B200_H
#define LOCKSTEP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LS_ABI_VERSION 3

/* ---- status codes ---------------------------------------------------------- */
enum {
  LS_OK = 0,
  LS_EINVAL = -1,   /* bad argument / malformed program            -> ValueError   */
  LS_ECUDA = -2,    /* CUDA failure or no device                   -> DeviceError  */
  LS_ENOMEM = -3,   /* device allocation failed                    -> DeviceError  */
};

/* ---- run outcome (ls_status.kind) -------------------------------------------- */
enum {
  LS_RUN_HALTED = 0,       /* every lane reached the halt block                   */
  LS_RUN_PAUSED = 1,       /* step budget of this call used, lanes still live     */
  LS_RUN_OVERFLOW = 2,     /* StackOverflow  (errors.py:54)                        */
  LS_RUN_UNDERFLOW = 3,    /* StackUnderflow (errors.py:58)                        */
  LS_RUN_STEP_LIMIT = 4,   /* StepLimitExceeded (errors.py:62)                     */
};

/* ---- storage classes (compiler.classify_variables) ----------------------------- */
enum { LS_STACKED = 0, LS_REGISTER = 1, LS_TEMPORARY = 2 };

/* ---- lane kinds (runtime.VType.kind) ---------------------------------------- */
enum { LS_F64 = 0, LS_I64 = 1, LS_BOOL = 2 };

/* ---- op actions (ir.Push / ir.Update / ir.Pop) ----------------------------- */
enum { LS_PUSH = 0, LS_UPDATE = 1, LS_POP = 2 };

/* ---- terminators (ir.FlatJump / FlatBranch / PushJump / FlatReturn) --------- */
enum { LS_JUMP = 0, LS_BRANCH = 1, LS_PUSHJUMP = 2, LS_RETURN = 3 };

/* ---- primitive opcodes (runtime.OPCODES) -------------------------------------- */
enum ls_opcode {
  LS_OP_NONE = 0,
  LS_OP_CONST = 1, LS_OP_ID = 2,
  LS_OP_ADD = 3, LS_OP_SUB = 4, LS_OP_MUL = 5, LS_OP_DIV = 6, LS_OP_MIN = 7, LS_OP_MAX = 8,
  LS_OP_LE = 9, LS_OP_LT = 10, LS_OP_EQ = 11,
  LS_OP_AND = 12, LS_OP_OR = 13, LS_OP_NOT = 14,
  LS_OP_NEG = 15, LS_OP_ABS = 16,
  LS_OP_SQRT = 17, LS_OP_EXP = 18, LS_OP_LOG = 19, LS_OP_SIN = 20, LS_OP_COS = 21,
  LS_OP_FLOOR = 22,
  LS_OP_SELECT = 23, LS_OP_DOT = 24, LS_OP_AXPY = 25,
  LS_OP_VGET = 26, LS_OP_VSTORE = 27, LS_OP_VCAT = 28, LS_OP_VFILL = 29, LS_OP_VSLICE = 30,
  LS_OP_RNG = 31,
  LS_OP_LOGPDF = 32, LS_OP_GRAD = 33,
  /* fused superblock: the whole leapfrog function (workloads.py:461-472)
     executed run-to-return for every selected lane; see DESIGN.md */
  LS_OP_LEAPFROG = 64,
  /* push that only allocates the new top slot: a caller save whose copy is never
     read (lowering.dead_saves); overflow-checked like any push */
  LS_OP_ALLOC = 65,
  /* fused momentum draw: the whole draw_normals(key, c) function of NUTS-lite
     (k Box-Muller normals from counters c+0.., then c + 2*ceil(k/2)) per lane;
     imm0 = k, imm1 = ceil(k/2); see lowering.match_normals */
  LS_OP_NORMALS = 66,
};

/* ---- target kinds (workloads.correlated_gaussian / logistic_regression) ------ */
enum { LS_TARGET_GAUSSIAN = 1, LS_TARGET_LOGREG = 2 };

/* ---- schedule rules ------------------------------------------------------------ */
enum {
  LS_SCHED_MIN_PC = 0,          /* reference rule: lowest populated block (pc_vm.py:306-311) */
  LS_SCHED_MOST_POPULATED = 1,  /* paper's throughput rule: block with most live lanes        */
  LS_SCHED_LOCAL = 2,           /* Alg. 1 local-static batching (reference local_exec.run_local):
                                   the deepest activation runs first, return landing pads first
                                   within it, then the lowest block (keys from the host)        */
  LS_SCHED_PRIORITY = 3,        /* least host-given block key (ls_machine_set_block_keys), e.g.
                                   reverse post-order with contraction blocks deferred          */
};

/* One flat op (ir.Push/Update/Pop). */
typedef struct {
  int32_t opcode;   /* enum ls_opcode; LS_OP_NONE for a pop                    */
  int32_t action;   /* LS_PUSH / LS_UPDATE / LS_POP                             */
  int32_t out;      /* output var (or popped var)                               */
  int32_t nin;      /* number of inputs                                         */
  int32_t in[3];    /* input vars                                               */
  int32_t kind;     /* lane kind of the first input (polymorphic arithmetic)   */
  int32_t width;    /* output width in words (1 for scalars)                   */
  int32_t imm0;     /* vfill width / vslice lo / target slot / leapfrog steps  */
  int32_t imm1;     /* vslice hi / leapfrog: var of q                          */
  int32_t imm2;     /* leapfrog: var of p                                       */
  int64_t bits;     /* const payload (f64 bits or i64)                          */
} ls_op;

/* One flat block. */
typedef struct {
  int32_t op_begin;
  int32_t op_count;
  int32_t term;     /* LS_JUMP / LS_BRANCH / LS_PUSHJUMP / LS_RETURN */
  int32_t a;        /* jump target, branch true target, pushjump jump_to     */
  int32_t b;        /* branch false target, pushjump return_to               */
  int32_t cond;     /* branch condition var                                   */
  int32_t grads;    /* grad-kernel invocations per lane in this block         */
  int32_t pad;
} ls_block;

/* One variable. */
typedef struct {
  int32_t cls;      /* LS_STACKED / LS_REGISTER / LS_TEMPORARY */
  int32_t kind;     /* LS_F64 / LS_I64 / LS_BOOL               */
  int32_t width;    /* words per lane (>= 1)                    */
  int32_t sp;       /* stack-pointer row for stacked vars, -1 otherwise */
  int32_t row;      /* first workspace row (non-stacked vars; views may share rows) */
  int32_t pad;
} ls_var;

typedef struct {
  const ls_block* blocks; int32_t n_blocks;
  const ls_op* ops;       int32_t n_ops;
  const ls_var* vars;     int32_t n_vars;
  int32_t entry;
  const int32_t* inputs;  int32_t n_inputs;
  int32_t output;
  int32_t flat_rows;      /* per-lane rows of all non-stacked storage (stacks follow) */
} ls_program_desc;

typedef struct {
  int32_t sched;          /* LS_SCHED_*                                               */
  int32_t lanes_per_cta;  /* lanes one VM group (CTA) schedules together; 0 = all Z
                             lanes in one group (exact reference schedule; Z <= 1024) */
  int32_t ctas;           /* persistent CTAs; 0 = one wave over all SMs               */
  int32_t trace;          /* record (block, active) per step (single group only)      */
  int32_t exact_logpdf;   /* 1: numpy einsum summation order; 0: fused fast form      */
  int32_t lane_trace_cap; /* >0: record each chain's block sequence (first cap steps) */
  int32_t warp_groups;    /* 1: throughput engine — every warp is a 32-lane group with
                             DMMA target contractions and fused superblocks; `ctas`
                             then caps the groups at 4 x ctas */
  int32_t flags;          /* LS_MF_* bits                                             */
  int32_t group_trace_cap; /* warp engine, >0: every group records its first cap steps
                             (block, active lanes) — the reference's per-step schedule
                             trace (metrics.py:36-41) per 32-lane group             */
} ls_machine_opts;

/* ls_machine_opts.flags */
#define LS_MF_FP32 2      /* warp engine, fp32 arm: fused leapfrogs in float32 on the tensor cores
                             (tcgen05 kind::tf32, 3xTF32 split); the warps of a warpgroup meet
                             at each superblock and contract their chains together (gaussian
                             targets, d <= 128) */
#define LS_MF_NO_STAGE 1  /* warp engine: read target matrices from global memory
                             instead of a per-CTA shared-memory copy */

typedef struct {
  int32_t kind;           /* LS_RUN_*                                          */
  int32_t var;            /* faulting variable (-1 = the pc stack)             */
  int64_t lane;           /* faulting lane (lowest index)                      */
  int32_t block;          /* block executing when the fault hit                */
  int32_t pad;
  int64_t steps;          /* steps executed so far (max over groups)           */
  int64_t useful_grads;   /* sum over steps of active lanes x grad invocations */
  int64_t launched_grads; /* sum over steps of group lanes x grad invocations  */
  double kernel_ms;       /* CUDA-event time of this call's VM launch, on the machine's stream */
  int64_t launches;       /* VM kernel launches issued by this machine so far  */
} ls_status;

typedef struct ls_program ls_program;
typedef struct ls_machine ls_machine;

int ls_abi_version(void);
const char* ls_last_error(void);
int ls_device_count(int32_t* n);
/* Select the CUDA device later ls_program_create / ls_machine_create calls of this host
   thread allocate on (one process per GPU: rank r passes its LOCAL_RANK). Programs and
   machines remember their device; every later call on them runs there. */
int ls_set_device(int32_t device);

int ls_program_create(const ls_program_desc* desc, ls_program** out);
/* Bind target slot `slot`: gaussian params = P (dim x dim, row-major) and
   `norm`; logistic params = sx (n x dim, row-major), norm unused. */
int ls_program_bind_target(ls_program* p, int32_t slot, int32_t kind, int32_t dim,
                           int32_t n, const double* params, double norm);
int ls_program_destroy(ls_program* p);

int ls_machine_create(ls_program* p, int64_t z, int32_t depth,
                      const ls_machine_opts* opts, ls_machine** out);
/* input `idx` of the program, host array of z * width words (lane-major) */
int ls_machine_set_input(ls_machine* m, int32_t idx, const void* host, int64_t bytes);
/* rewind a machine to its freshly-seeded state (inputs kept), without reallocating */
int ls_machine_reset(ls_machine* m);
/* keyed schedule rules (min_pc, local, priority): the least keys[b] among live lanes' blocks
   runs next; bits 0..15 of keys[b] must equal b (the local rule uses bits 0..23). Default: keys[b] = b (the reference's
   min-pc rule, pc_vm.py:306-311). Replaces the step selection of pc_vm.step. */
int ls_machine_set_block_keys(ls_machine* m, const uint32_t* keys, int32_t n_blocks);
/* same, from device memory (e.g. a torch CUDA tensor) */
int ls_machine_set_input_device(ls_machine* m, int32_t idx, const void* dev, int64_t bytes);
/* Execute up to max_steps steps per group (<0: unbounded). Returns LS_OK and
   fills *st; faults are reported in st->kind, not as an error code. */
int ls_run(ls_machine* m, int64_t max_steps, ls_status* st);
int ls_read_output(ls_machine* m, void* host, int64_t bytes);
/* warp engine: have the kernel write output rows straight into a page-locked buffer
   from ls_host_alloc (overlapping the transfer with the run; host = NULL reverts to
   device memory); ls_read_output from that buffer is then only a synchronisation */
int ls_machine_set_output_host(ls_machine* m, void* host, int64_t bytes);
/* device pointer of the z x width output (valid until destroy) */
int ls_output_device(ls_machine* m, void** dev);
/* device-to-device copy of the output's first bytes / (width * 8) rows (e.g. into a torch
   CUDA tensor for NCCL diagnostics) */
int ls_copy_output_device(ls_machine* m, void* dev_dst, int64_t bytes);
/* drain recorded (block, active) step pairs; *n = number written */
int ls_trace_fetch(ls_machine* m, int32_t* blocks, int32_t* active, int64_t cap, int64_t* n);
/* per-block totals over all groups: steps executed and sum of active lanes */
int ls_block_totals(ls_machine* m, int64_t* steps, int64_t* active);
/* warp engine: SM clock cycles each block's steps took, summed over groups (a
   cycle-weighted profile of the program, complementary to ncu stall sampling) */
int ls_block_cycles(ls_machine* m, int64_t* cycles);
/* observer access (single-group machines): all `depth` slots of a var as
   host array [slots][z][width]; pointers as [z] int64 (stacked vars / -1 = pc) */
int ls_read_var(ls_machine* m, int32_t var, void* host, int64_t bytes);
int ls_read_pointers(ls_machine* m, int32_t var, int64_t* host, int64_t z);
/* the pc stack of a single-group machine as host [depth+1][z] int32 */
int ls_read_pc_stack(ls_machine* m, int32_t* host, int64_t count);
/* per-chain block sequences: blocks [z][cap], lens [z] (a len > cap was truncated) */
int ls_lane_trace_fetch(ls_machine* m, int32_t* blocks, int32_t* lens, int64_t cap);
/* warp engine step records per group (reference ScheduleTrace.record, metrics.py:36-37, one
   trace per 32-lane group): recs [groups][cap] = block | active << 16, a paired step (two
   blocks of identical code on different variables) as two records; lens [groups] (> cap:
   truncated). Needs group_trace_cap > 0 at create; groups from ls_machine_info. */
int ls_group_trace_fetch(ls_machine* m, int32_t* recs, int32_t* lens, int64_t cap);
int ls_machine_sync(ls_machine* m);
/* where and how a machine runs: CUDA device, schedule groups, lanes per group */
int ls_machine_info(const ls_machine* m, int32_t* device, int32_t* groups, int32_t* lanes_per_group);
int ls_machine_destroy(ls_machine* m);

/* page-locked (and device-mapped) host buffers: ls_read_output into one is a direct
   DMA, and ls_machine_set_output_host accepts them (_native.HostPool) */
int ls_host_alloc(int64_t bytes, void** host);
int ls_host_free(void* host);

/* runtime.rng_uniform over n lanes (keys/counters as int64 after numpy's astype) */
int ls_rng_uniform(const int64_t* key, const int64_t* counter, int64_t n, double* out);
/* evaluate a target's logpdf (which=0) or grad (which=1) on z points x[z][dim] */
int ls_target_eval(int32_t kind, int32_t which, int32_t dim, int32_t n, const double* params,
                   double norm, const double* x, int64_t z, double* out);

#ifdef __cplusplus
}
#endif
#endif /* LOCKSTEP_B200_H */
