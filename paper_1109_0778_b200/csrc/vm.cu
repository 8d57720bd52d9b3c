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
// division by zero and out-of-range loads raise the trap flag (TrapError on the host).
#include <algorithm>

#include "common.cuh"
#include "../../include/dlx_vm.h"

namespace dlx {

union Reg {
  long long i;
  double d;
};

constexpr int kVmThreads = 256;

__device__ __forceinline__ void vm_exec(const dlx_vm_instr* __restrict__ code, int begin, int end,
                                        Reg* r, long long idx, const dlx_vm_loop* L, int* trap) {
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
          atomicOr(trap, 2);
          d.i = 0;
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
          atomicOr(trap, 1);
          d.i = 0;
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
      default: atomicOr(trap, 4); break;
    }
  }
}

__global__ void __launch_bounds__(kVmThreads)
vm_loop_kernel(const dlx_vm_instr* __restrict__ code, dlx_vm_loop L, Reg* __restrict__ parts,
               int* __restrict__ trap) {
  __shared__ dlx_vm_instr code_s[DLX_VM_MAX_CODE];
  __shared__ Reg red_s[kVmThreads / 32][DLX_VM_MAX_ELEMS];
  for (int e = threadIdx.x; e < L.ncode; e += kVmThreads) code_s[e] = code[e];
  __syncthreads();
  Reg acc[DLX_VM_MAX_ELEMS];
  for (int e = 0; e < L.nelems; ++e) acc[e].i = L.elem[e].zero;
  Reg r[DLX_VM_MAX_REGS];
  const long long T = static_cast<long long>(gridDim.x) * kVmThreads;
  for (long long i = static_cast<long long>(blockIdx.x) * kVmThreads + threadIdx.x; i < L.range; i += T) {
    vm_exec(code_s, 0, L.body_end, r, i, &L, trap);
    for (int e = 0; e < L.nelems; ++e) {
      const dlx_vm_elem& el = L.elem[e];
      if (el.cond_end > el.cond_begin) {
        vm_exec(code_s, el.cond_begin, el.cond_end, r, i, &L, trap);
        if (!r[el.cond_reg].i) continue;
      }
      vm_exec(code_s, el.value_begin, el.value_end, r, i, &L, trap);
      const Reg v = r[el.value_reg];
      if (el.kind == DLX_VM_COLLECT) {
        if (el.ty == DLX_VM_F64) static_cast<double*>(el.out)[i] = v.d;
        else if (el.ty == DLX_VM_I64) static_cast<long long*>(el.out)[i] = v.i;
        else static_cast<unsigned char*>(el.out)[i] = static_cast<unsigned char>(v.i != 0);
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
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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

// fold CTA partials in ascending order (the zero is already folded into every partial
// except the first, so fold partial 0 then combine the rest)
__global__ void vm_final_kernel(const Reg* __restrict__ parts, int nparts, dlx_vm_loop L,
                                long long* __restrict__ out) {
  const int e = threadIdx.x;
  if (e >= L.nelems || L.elem[e].kind != DLX_VM_REDUCE) return;
  const dlx_vm_elem& el = L.elem[e];
  Reg v = parts[e];
  for (int p = 1; p < nparts; ++p) {
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
  return static_cast<size_t>(vm_grid(range)) * DLX_VM_MAX_ELEMS * sizeof(Reg) + 1024;
}

int dlx_vm_run_loop(const dlx_vm_instr* d_code, const dlx_vm_loop* h_loop, int64_t* d_results,
                    int* d_trap, void* d_workspace, size_t workspace_bytes, dlx_stream_t stream) {
  DLX_REQUIRE(h_loop && d_code && d_trap && d_results, DLX_ERR_ARG, "vm: null argument");
  const dlx_vm_loop& L = *h_loop;
  DLX_REQUIRE(L.ncode <= DLX_VM_MAX_CODE && L.nelems <= DLX_VM_MAX_ELEMS && L.range >= 0,
              DLX_ERR_GENERATION, "GenerationFailed: multiloop exceeds the generic kernel's plan");
  if (L.range == 0) {
    // every reduce keeps its zero: the host layer binds zeros without a launch
    return DLX_OK;
  }
  const int grid = vm_grid(L.range);
  DLX_REQUIRE(d_workspace && workspace_bytes >= static_cast<size_t>(grid) * DLX_VM_MAX_ELEMS * sizeof(Reg),
              DLX_ERR_ARG, "vm: workspace too small");
  Reg* parts = static_cast<Reg*>(d_workspace);
  vm_loop_kernel<<<grid, kVmThreads, 0, stream>>>(d_code, L, parts, d_trap);
  DLX_LAUNCHED("vm_loop_kernel");
  vm_final_kernel<<<1, DLX_VM_MAX_ELEMS, 0, stream>>>(parts, grid, L, reinterpret_cast<long long*>(d_results));
  DLX_LAUNCHED("vm_final_kernel");
  return DLX_OK;
}

}  // extern "C"
