/*
 * dlx_vm.h — C ABI of the generic multiloop kernel (paper_1109_0778_b200/csrc/vm.cu).
 *
 * Replaces emit_parallel_loop's per-index lowering (proj/src/codegen.cpp:345-433) for fused
 * loops outside the specialised families: the loop's live elems (LoopElem, node.hpp:60-74)
 * are compiled by the host executor into a register bytecode over element loads, scalar
 * arithmetic (the Op set of node.hpp:15-27, plus the MathExp extension), Select for
 * IfThenElse values, cond guards, and a Plus / Times combine.  One launch runs the whole
 * multiloop; dense collects are written in place, reduce results land in d_results[elem]
 * (64-bit: int64 or the bits of an fp64).
 */
#ifndef DLX_VM_H_
#define DLX_VM_H_

#include <stddef.h>
#include <stdint.h>

#include "dlx.h"

#ifdef __cplusplus
extern "C" {
#endif

#define DLX_VM_MAX_CODE 512
#define DLX_VM_MAX_ELEMS 16
#define DLX_VM_MAX_REGS 48
#define DLX_VM_MAX_VECS 8

enum dlx_vm_op {
  DLX_VM_CONST = 0, /* dst = imm (64-bit pattern) */
  DLX_VM_IDX,       /* dst = loop index */
  DLX_VM_LOAD,      /* dst = vec[aux][reg a]  (bounds-checked: DLX_VM_TRAP_BOUNDS) */
  DLX_VM_ADD_I, DLX_VM_SUB_I, DLX_VM_MUL_I, DLX_VM_DIV_I, /* int64, wraparound; /0 -> DLX_VM_TRAP_DIV0 */
  DLX_VM_ADD_D, DLX_VM_SUB_D, DLX_VM_MUL_D, DLX_VM_DIV_D, /* fp64, round-to-nearest, no FMA */
  DLX_VM_LT_I, DLX_VM_LT_D, DLX_VM_EQ_I, DLX_VM_EQ_D,
  DLX_VM_AND, DLX_VM_OR, DLX_VM_NOT,
  DLX_VM_ABS_I, DLX_VM_ABS_D, DLX_VM_SQRT, DLX_VM_EXP, DLX_VM_TODBL,
  DLX_VM_SEL        /* dst = reg[imm] ? a : b */
};

enum { DLX_VM_I64 = 0, DLX_VM_F64 = 1, DLX_VM_BOOL = 2 };
/* DLX_VM_APPEND: filter-collect (LoopElem.append, codegen.cpp:357-360 / 404-405): the values of
 * the indices whose cond holds, appended in index order; d_results[elem] receives the length. */
enum { DLX_VM_COLLECT = 0, DLX_VM_REDUCE = 1, DLX_VM_APPEND = 2 };
enum { DLX_VM_COMBINE_ADD = 0, DLX_VM_COMBINE_MUL = 1 };

typedef struct {
  uint8_t op, dst, a, b;
  int32_t aux;
  int64_t imm;
} dlx_vm_instr;

typedef struct {
  int32_t kind;        /* DLX_VM_COLLECT / DLX_VM_REDUCE */
  int32_t ty;          /* element type */
  int32_t combine;     /* reduce: DLX_VM_COMBINE_* */
  int32_t cond_begin, cond_end, cond_reg;   /* empty range = no guard */
  int32_t value_begin, value_end, value_reg;
  int64_t zero;        /* reduce identity (bits) */
  void* out;           /* collect / append: device output vector with room for `range` elements */
} dlx_vm_elem;

typedef struct {
  int64_t range;
  int32_t ncode, body_end, nelems, nvecs;
  const void* vec[DLX_VM_MAX_VECS];
  int64_t vec_len[DLX_VM_MAX_VECS];
  int32_t vec_kind[DLX_VM_MAX_VECS];
  dlx_vm_elem elem[DLX_VM_MAX_ELEMS];
} dlx_vm_loop;

/* workspace for one dlx_vm_run_loop of this range (per-CTA reduce partials, and for append
 * elems the per-CTA counts and offsets) */
size_t dlx_vm_workspace_bytes(int64_t range);
/* d_code: ncode instructions in device memory; d_results: DLX_VM_MAX_ELEMS 64-bit slots;
 * d_trap: one device uint64 the caller sets to UINT64_MAX; it ends as the minimum over trapped
 * indices of (index << 2 | DLX_VM_TRAP_*), i.e. the first trap sequential execution meets
 * (UINT64_MAX: none). */
#define DLX_VM_TRAP_DIV0 1   /* Int division by zero (TrapDivByZero) */
#define DLX_VM_TRAP_BOUNDS 2 /* element load out of range (TrapIndexOutOfBounds) */
#define DLX_VM_TRAP_BADOP 3  /* unknown instruction (GenerationFailed) */
int dlx_vm_run_loop(const dlx_vm_instr* d_code, const dlx_vm_loop* h_loop, int64_t* d_results,
                    uint64_t* d_trap, void* d_workspace, size_t workspace_bytes, dlx_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* DLX_VM_H_ */
