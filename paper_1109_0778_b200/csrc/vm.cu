// vm.cu — the generic multiloop kernel: any fused loop whose live elems are Collect (dense)
// or Reduce (+ / * combine) over scalar expression DAGs of element loads at affine indices,
// with optional cond guards ("generic elem-block lowering").  The C++
// executor (program.cpp) compiles each elem's blocks into a register bytecode; this kernel
// runs the whole multiloop in one pass, one thread per index in a grid-stride loop, exactly
// in emit_parallel_loop's per-index order (proj/src/codegen.cpp:382-426): shared body-scope
// code, then per elem `if (cond) { collect store | acc = combine(acc, elem) }`.
// Reduce slots fold per thread, then warp / CTA trees, then the deterministic combine of
// per-CTA partials (combine.cu).  fp64 arithmetic uses explicit _rn intrinsics (no FMA
// contraction) so collects are bit-identical to the reference; Int arithmetic wraps; Int
// division by zero and out-of-range loads record the first trap in index order (TrapError on the host).
// Filter-collect (append) elems make the launch order-preserving: a count pass over contiguous
// per-CTA index ranges, an exclusive scan of the per-CTA counts, then the main pass writes each
// CTA's selected values at its offset with a block-wide ballot scan per 256-index step, so the
// output is exactly the reference's builder contents in index order.
#include <algorithm>

#include "common.cuh"
#include "../../include/dlx_vm.h"

namespace dlx {

union Reg {
  long long i;
  double d;
};

constexpr int kVmThreads = 256;

// record a trap of index idx: the word keeps the minimum (idx << 2 | kind), i.e. the first trap
// in index order, as sequential interpret stops at it (codegen.cpp:391-425: indices ascend, and
// within an index the body and the elems run in program order)
__device__ __forceinline__ void vm_trap(unsigned long long* trap, long long idx, int kind) {
  atomicMin(trap, (static_cast<unsigned long long>(idx) << 2) | static_cast<unsigned long long>(kind));
}

// runs code[begin, end) for index idx; false once it trapped (the caller then abandons the index,
// so no later statement or elem of it runs and no second trap of it is recorded)
__device__ __forceinline__ bool vm_exec(const dlx_vm_instr* __restrict__ code, int begin, int end,
                                        Reg* r, long long idx, const dlx_vm_loop* L,
                                        unsigned long long* trap) {
  for (int pc = begin; pc < end; ++pc) {
    const dlx_vm_instr in = code[pc];
    Reg& d = r[in.dst];
    const Reg a = r[in.a], b = r[in.b];
    switch (in.op) {
      case DLX_VM_CONST: d.i = in.imm; break;
      case DLX_VM_IDX: d.i = idx; break;
      case DLX_VM_LOAD: {
        const long long k = a.i;
        if (k < 0 || k >= L->vec_len[in.aux]) {
          vm_trap(trap, idx, DLX_VM_TRAP_BOUNDS);
          return false;
        } else if (L->vec_kind[in.aux] == DLX_VM_F64) {
          d.d = static_cast<const double*>(L->vec[in.aux])[k];
        } else if (L->vec_kind[in.aux] == DLX_VM_I64) {
          d.i = static_cast<const long long*>(L->vec[in.aux])[k];
        } else {
          d.i = static_cast<const unsigned char*>(L->vec[in.aux])[k];
        }
        break;
      }
      case DLX_VM_ADD_I: d.i = static_cast<long long>(static_cast<unsigned long long>(a.i) + static_cast<unsigned long long>(b.i)); break;
      case DLX_VM_SUB_I: d.i = static_cast<long long>(static_cast<unsigned long long>(a.i) - static_cast<unsigned long long>(b.i)); break;
      case DLX_VM_MUL_I: d.i = static_cast<long long>(static_cast<unsigned long long>(a.i) * static_cast<unsigned long long>(b.i)); break;
      case DLX_VM_DIV_I:
        if (b.i == 0) {
          vm_trap(trap, idx, DLX_VM_TRAP_DIV0);
          return false;
        } else {
          d.i = (a.i == LLONG_MIN && b.i == -1) ? a.i : a.i / b.i;
        }
        break;
      case DLX_VM_ADD_D: d.d = __dadd_rn(a.d, b.d); break;
      case DLX_VM_SUB_D: d.d = __dsub_rn(a.d, b.d); break;
      case DLX_VM_MUL_D: d.d = __dmul_rn(a.d, b.d); break;
      case DLX_VM_DIV_D: d.d = __ddiv_rn(a.d, b.d); break;
      case DLX_VM_LT_I: d.i = a.i < b.i; break;
      case DLX_VM_LT_D: d.i = a.d < b.d; break;
      case DLX_VM_EQ_I: d.i = a.i == b.i; break;
      case DLX_VM_EQ_D: d.i = a.d == b.d; break;
      case DLX_VM_AND: d.i = (a.i != 0) && (b.i != 0); break;
      case DLX_VM_OR: d.i = (a.i != 0) || (b.i != 0); break;
      case DLX_VM_NOT: d.i = a.i == 0; break;
      case DLX_VM_ABS_I: d.i = a.i < 0 ? static_cast<long long>(0ull - static_cast<unsigned long long>(a.i)) : a.i; break;
      case DLX_VM_ABS_D: d.d = fabs(a.d); break;
      case DLX_VM_SQRT: d.d = __dsqrt_rn(a.d); break;
      case DLX_VM_EXP: d.d = exp(a.d); break;
      case DLX_VM_TODBL: d.d = static_cast<double>(a.i); break;
      case DLX_VM_SEL: d = r[in.imm].i ? a : b; break;  // imm holds the condition register
      default: vm_trap(trap, idx, DLX_VM_TRAP_BADOP); return false;
    }
  }
  return true;
}

__device__ __forceinline__ void vm_store(const dlx_vm_elem& el, long long at, Reg v) {
  if (el.ty == DLX_VM_F64) static_cast<double*>(el.out)[at] = v.d;
  else if (el.ty == DLX_VM_I64) static_cast<long long*>(el.out)[at] = v.i;
  else static_cast<unsigned char*>(el.out)[at] = static_cast<unsigned char>(v.i != 0);
}

// contiguous index range of CTA b when the loop has append elems
__device__ __forceinline__ void vm_chunk(long long range, long long chunk, long long& lo, long long& hi) {
  lo = static_cast<long long>(blockIdx.x) * chunk;
  hi = lo + chunk < range ? lo + chunk : range;
}

// count pass: how many indices of this CTA's range each append elem selects
__global__ void __launch_bounds__(kVmThreads)
vm_count_kernel(const dlx_vm_instr* __restrict__ code, dlx_vm_loop L, long long chunk,
                long long* __restrict__ counts, unsigned long long* __restrict__ trap) {
  __shared__ dlx_vm_instr code_s[DLX_VM_MAX_CODE];
  __shared__ long long cnt_s[DLX_VM_MAX_ELEMS];
  for (int e = threadIdx.x; e < L.ncode; e += kVmThreads) code_s[e] = code[e];
  if (threadIdx.x < DLX_VM_MAX_ELEMS) cnt_s[threadIdx.x] = 0;
  __syncthreads();
  long long lo, hi;
  vm_chunk(L.range, chunk, lo, hi);
  Reg r[DLX_VM_MAX_REGS];
  int my[DLX_VM_MAX_ELEMS];
  for (int e = 0; e < L.nelems; ++e) my[e] = 0;
  for (long long i = lo + threadIdx.x; i < hi; i += kVmThreads) {
    if (!vm_exec(code_s, 0, L.body_end, r, i, &L, trap)) continue;
    for (int e = 0; e < L.nelems; ++e) {
      const dlx_vm_elem& el = L.elem[e];
      if (el.kind != DLX_VM_APPEND) continue;
      bool take = true;
      if (el.cond_end > el.cond_begin) {
        if (!vm_exec(code_s, el.cond_begin, el.cond_end, r, i, &L, trap)) break;
        take = r[el.cond_reg].i != 0;
      }
      my[e] += take;
    }
  }
  for (int e = 0; e < L.nelems; ++e) {
    if (L.elem[e].kind != DLX_VM_APPEND) continue;
    int v = my[e];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt_s[e]), static_cast<unsigned long long>(v));
  }
  __syncthreads();
  if (threadIdx.x < L.nelems) counts[static_cast<size_t>(blockIdx.x) * DLX_VM_MAX_ELEMS + threadIdx.x] = cnt_s[threadIdx.x];
}

// exclusive scan of the per-CTA counts (ascending CTA = ascending index ranges) -> offsets,
// and the total = the appended vector's length
__global__ void vm_scan_kernel(const long long* __restrict__ counts, int nblocks, dlx_vm_loop L,
                               long long* __restrict__ offsets, long long* __restrict__ out) {
  const int e = threadIdx.x;
  if (e >= L.nelems || L.elem[e].kind != DLX_VM_APPEND) return;
  long long run = 0;
  for (int b = 0; b < nblocks; ++b) {
    offsets[static_cast<size_t>(b) * DLX_VM_MAX_ELEMS + e] = run;
    run += counts[static_cast<size_t>(b) * DLX_VM_MAX_ELEMS + e];
  }
  out[e] = run;
}

__global__ void __launch_bounds__(kVmThreads)
vm_loop_kernel(const dlx_vm_instr* __restrict__ code, dlx_vm_loop L, Reg* __restrict__ parts,
               unsigned long long* __restrict__ trap, long long chunk, const long long* __restrict__ offsets) {
  __shared__ dlx_vm_instr code_s[DLX_VM_MAX_CODE];
  __shared__ Reg red_s[kVmThreads / 32][DLX_VM_MAX_ELEMS];
  __shared__ int wsum_s[kVmThreads / 32];
  for (int e = threadIdx.x; e < L.ncode; e += kVmThreads) code_s[e] = code[e];
  __syncthreads();
  Reg acc[DLX_VM_MAX_ELEMS];
  long long run[DLX_VM_MAX_ELEMS];   // append: next output slot of this CTA
  for (int e = 0; e < L.nelems; ++e) {
    // start at the combine's identity (-0.0 / 0 / 1): the elem's `zero` is folded exactly once, by
    // vm_final_kernel, as in `var acc = zero; for i: acc = combine(acc, elem)` (codegen.cpp:367-369)
    const bool mul = L.elem[e].combine == DLX_VM_COMBINE_MUL;
    if (L.elem[e].ty == DLX_VM_F64) acc[e].d = mul ? 1.0 : -0.0;   // -0.0 + x == x for every x
    else acc[e].i = mul ? 1 : 0;
    run[e] = (chunk > 0 && L.elem[e].kind == DLX_VM_APPEND)
                 ? offsets[static_cast<size_t>(blockIdx.x) * DLX_VM_MAX_ELEMS + e] : 0;
  }
  Reg r[DLX_VM_MAX_REGS];
  // grid-stride without append elems; contiguous per-CTA ranges (all threads step together,
  // so the append scan stays in index order) with them
  long long i, stop, step;
  if (chunk > 0) {
    vm_chunk(L.range, chunk, i, stop);
    step = kVmThreads;
  } else {
    i = static_cast<long long>(blockIdx.x) * kVmThreads;
    stop = L.range;
    step = static_cast<long long>(gridDim.x) * kVmThreads;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (; i < stop; i += step) {
    const long long idx = i + threadIdx.x;
    bool live = idx < stop;
    if (live) live = vm_exec(code_s, 0, L.body_end, r, idx, &L, trap);
    for (int e = 0; e < L.nelems; ++e) {
      const dlx_vm_elem& el = L.elem[e];
      // a trapped index stays `live == false` for its remaining elems (the loop is abandoned
      // on the host anyway; every thread still reaches the append scans below)
      bool take = live;
      if (live && el.cond_end > el.cond_begin) {
        live = vm_exec(code_s, el.cond_begin, el.cond_end, r, idx, &L, trap);
        take = live && r[el.cond_reg].i != 0;
      }
      Reg v;
      v.i = 0;
      if (take) {
        live = vm_exec(code_s, el.value_begin, el.value_end, r, idx, &L, trap);
        take = live;
        v = r[el.value_reg];
      }
      if (el.kind == DLX_VM_APPEND) {   // block-uniform branch: every thread reaches the scan
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if (lane == 0) wsum_s[warp] = __popc(bal);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < kVmThreads / 32; ++w) {
          const int c = wsum_s[w];
          before += w < warp ? c : 0;
          total += c;
        }
        if (take) vm_store(el, run[e] + before + __popc(bal & ((1u << lane) - 1)), v);
        run[e] += total;
        __syncthreads();
        continue;
      }
      if (!take) continue;
      if (el.kind == DLX_VM_COLLECT) {
        vm_store(el, idx, v);
      } else if (el.ty == DLX_VM_F64) {
        acc[e].d = el.combine == DLX_VM_COMBINE_MUL ? __dmul_rn(acc[e].d, v.d) : __dadd_rn(acc[e].d, v.d);
      } else {
        acc[e].i = el.combine == DLX_VM_COMBINE_MUL
                       ? static_cast<long long>(static_cast<unsigned long long>(acc[e].i) * static_cast<unsigned long long>(v.i))
                       : static_cast<long long>(static_cast<unsigned long long>(acc[e].i) + static_cast<unsigned long long>(v.i));
      }
    }
  }
  // warp tree, then ascending-warp fold, per reduce elem
  for (int e = 0; e < L.nelems; ++e) {
    const dlx_vm_elem& el = L.elem[e];
    if (el.kind != DLX_VM_REDUCE) continue;
    Reg v = acc[e];
    for (int o = 16; o > 0; o >>= 1) {
      Reg w;
      w.i = __shfl_xor_sync(0xffffffffu, v.i, o);
      if (el.ty == DLX_VM_F64) v.d = el.combine == DLX_VM_COMBINE_MUL ? __dmul_rn(v.d, w.d) : __dadd_rn(v.d, w.d);
      else v.i = el.combine == DLX_VM_COMBINE_MUL ? v.i * w.i : v.i + w.i;
    }
    if (lane == 0) red_s[warp][e] = v;
  }
  __syncthreads();
  if (threadIdx.x < L.nelems) {
    const int e = threadIdx.x;
    const dlx_vm_elem& el = L.elem[e];
    if (el.kind == DLX_VM_REDUCE) {
      Reg v = red_s[0][e];
      for (int w = 1; w < kVmThreads / 32; ++w) {
        const Reg u = red_s[w][e];
        if (el.ty == DLX_VM_F64) v.d = el.combine == DLX_VM_COMBINE_MUL ? __dmul_rn(v.d, u.d) : __dadd_rn(v.d, u.d);
        else v.i = el.combine == DLX_VM_COMBINE_MUL ? v.i * u.i : v.i + u.i;
      }
      parts[static_cast<size_t>(blockIdx.x) * DLX_VM_MAX_ELEMS + e] = v;
    }
  }
}

// fold the elem's zero, then the CTA partials in ascending order (each partial started at the
// combine's identity, so the zero enters the result exactly once)
__global__ void vm_final_kernel(const Reg* __restrict__ parts, int nparts, dlx_vm_loop L,
                                long long* __restrict__ out) {
  const int e = threadIdx.x;
  if (e >= L.nelems || L.elem[e].kind != DLX_VM_REDUCE) return;
  const dlx_vm_elem& el = L.elem[e];
  Reg v;
  v.i = el.zero;
  for (int p = 0; p < nparts; ++p) {
    const Reg u = parts[static_cast<size_t>(p) * DLX_VM_MAX_ELEMS + e];
    if (el.ty == DLX_VM_F64) v.d = el.combine == DLX_VM_COMBINE_MUL ? __dmul_rn(v.d, u.d) : __dadd_rn(v.d, u.d);
    else v.i = el.combine == DLX_VM_COMBINE_MUL ? v.i * u.i : v.i + u.i;
  }
  out[e] = v.i;
}

static int vm_grid(long long range) {
  const long long need = (range + kVmThreads - 1) / kVmThreads;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(need, sm_count() * 4)));
}

}  // namespace dlx

using namespace dlx;

extern "C" {

size_t dlx_vm_workspace_bytes(int64_t range) {
  // reduce partials, append counts, append offsets
  return 3 * static_cast<size_t>(vm_grid(range)) * DLX_VM_MAX_ELEMS * sizeof(Reg) + 1024;
}

int dlx_vm_run_loop(const dlx_vm_instr* d_code, const dlx_vm_loop* h_loop, int64_t* d_results,
                    uint64_t* d_trap, void* d_workspace, size_t workspace_bytes, dlx_stream_t stream) {
  DLX_REQUIRE(h_loop && d_code && d_trap && d_results, DLX_ERR_ARG, "vm: null argument");
  const dlx_vm_loop& L = *h_loop;
  DLX_REQUIRE(L.ncode <= DLX_VM_MAX_CODE && L.nelems <= DLX_VM_MAX_ELEMS && L.range >= 0,
              DLX_ERR_GENERATION, "GenerationFailed: multiloop exceeds the generic kernel's plan");
  if (L.range == 0) {
    // every reduce keeps its zero: the host layer binds zeros without a launch
    return DLX_OK;
  }
  const int grid = vm_grid(L.range);
  DLX_REQUIRE(d_workspace && workspace_bytes >= 3 * static_cast<size_t>(grid) * DLX_VM_MAX_ELEMS * sizeof(Reg),
              DLX_ERR_ARG, "vm: workspace too small");
  bool append = false;
  for (int e = 0; e < L.nelems; ++e) append |= L.elem[e].kind == DLX_VM_APPEND;
  Reg* parts = static_cast<Reg*>(d_workspace);
  long long* counts = reinterpret_cast<long long*>(parts + static_cast<size_t>(grid) * DLX_VM_MAX_ELEMS);
  long long* offsets = counts + static_cast<size_t>(grid) * DLX_VM_MAX_ELEMS;
  long long chunk = 0;
  if (append) {
    chunk = (L.range + grid - 1) / grid;
    vm_count_kernel<<<grid, kVmThreads, 0, stream>>>(d_code, L, chunk, counts,
                                                     reinterpret_cast<unsigned long long*>(d_trap));
    DLX_LAUNCHED("vm_count_kernel");
    vm_scan_kernel<<<1, DLX_VM_MAX_ELEMS, 0, stream>>>(counts, grid, L, offsets,
                                                       reinterpret_cast<long long*>(d_results));
    DLX_LAUNCHED("vm_scan_kernel");
  }
  vm_loop_kernel<<<grid, kVmThreads, 0, stream>>>(d_code, L, parts, reinterpret_cast<unsigned long long*>(d_trap),
                                                  chunk, offsets);
  DLX_LAUNCHED("vm_loop_kernel");
  vm_final_kernel<<<1, DLX_VM_MAX_ELEMS, 0, stream>>>(parts, grid, L, reinterpret_cast<long long*>(d_results));
  DLX_LAUNCHED("vm_final_kernel");
  return DLX_OK;
}

}  // extern "C"
