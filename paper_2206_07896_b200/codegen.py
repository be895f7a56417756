"""CUDA code generation for arbitrary reference kernels.

The hand-written sm_100a kernels cover the registered routines.  Any other
kernel the reference can express arrives at `Runtime.launch` as an
`MpmdKernel` (transform.py:109-221) whose sections still hold the validated,
type-annotated AST (validate.py:187-301 sets `.ty` on every expression).
This module turns that AST into a CUDA kernel with the reference's exact
semantics, which libbfgpu.so compiles with NVRTC for sm_100a and registers
under a fingerprint key (bf_jit_register):

  * a CTA is one logical block (blockDim.x*y*z <= 1024 threads); a grid-stride
    loop walks the fetched block range; sections run in order with
    __syncthreads at every barrier (the lockstep chunks of
    executor.run_reference, executor.py:422-489, for race-free code);
  * i32/i64 arithmetic wraps after every operator; / and % truncate toward
    zero and trap on 0 (interp.py:45-91); float math is IEEE double and
    rounds to f32 only when stored into an f32 array (arena.py:111-116);
    f32 locals and params hold doubles (interp.py:94-99, hostprog.py:153);
  * every array access is bounds-checked (Trap OutOfBounds), sqrt of a
    negative value and float division by zero trap (interp.py:68-70,147-149);
  * shared arrays are zeroed at block entry (executor.py:441-453);
  * atomics: add / cas with the reference's coerce rules (executor.py:184-214)
    — f32 adds round once, RN32(old + operand), via a CAS loop;
  * warp mode: shfl_down / vote_* over logical warps of `warp_size` lanes
    with the reference's clamp (interp.py:256-297), exchanged through shared
    memory so any warp size works.

Compiled with -fmad=false: no FMA contraction anywhere.
"""

from __future__ import annotations

import hashlib
import struct
from typing import Optional

_CTYPE = {"i32": "int", "i64": "long long", "f32": "double", "f64": "double"}
_MTYPE = {"i32": "int", "i64": "long long", "f32": "float", "f64": "double"}  # memory element
_SIZE = {"i32": 4, "i64": 8, "f32": 4, "f64": 8}
_TRAP = {"OutOfBounds": 1, "DivByZero": 2, "TypeFault": 3, "NonUniformTrip": 4}
WARP_INTRINSICS = ("shfl_down", "vote_any", "vote_all")


class CodegenError(Exception):
    pass


def _cls(node) -> str:
    return type(node).__name__


def _float_lit(v: float) -> str:
    if v != v:
        return "__longlong_as_double(0x7ff8000000000000LL)"
    if v in (float("inf"), float("-inf")):
        return "(1.0/0.0)" if v > 0 else "(-1.0/0.0)"
    return f"__longlong_as_double({struct.unpack('<q', struct.pack('<d', v))[0]}LL)"


PRELUDE = r"""
struct BfJitGeom {
  int gx, gy, gz, bx, by, bz;
  long long first, count;
  long long dyn_elems;
  int* fault;  // {kind, pad, block(lo, hi), task(lo, hi), host flag pointer}
  unsigned long long task;
  int warp_size;
  // device-side fetching (null dcur: the grid strides over [first, first + count));
  // the fetches are split into 8 sub-ranges with a claim counter each, zeroed
  // at launch (bf_internal.h DevFetch)
  unsigned long long* dcur;    // the worker's 8 claim counters
  unsigned long long* dstats;  // per worker slot: claims, blocks executed
  int* dexec;                  // KernelTask.executed by absolute block (nullable)
  long long nfetch, grain;
  int dslots;
};
// thread 0's claim of the next fetch (cursor: sub-range and sub-ranges tried;
// the CTA's claims are counted in a register and flushed once at the end)
__device__ __forceinline__ long long bf_claim(const BfJitGeom& G, int& sub, int& tried, unsigned long long& nclaims) {
  while (tried < 8) {
    const long long lo = (G.nfetch * sub) / 8, n = (G.nfetch * (sub + 1)) / 8 - lo;
    const long long f = (long long)atomicAdd(G.dcur + sub, 1ull);
    if (f < n) {
      nclaims++;
      return lo + f;
    }
    sub = (sub + 1) %% 8;
    tried++;
  }
  return G.nfetch;
}
__device__ __forceinline__ long long bf_take(long long mine) {
  __shared__ long long s_claim;
  __syncthreads();
  if (threadIdx.x == 0) s_claim = mine;
  __syncthreads();
  return s_claim;
}
struct BfJitArgs { long long w[%(nw)d]; };

// a trap records the first fault and stops the trapping thread's side
// effects (stores, atomics, loops): the reference aborts the block at the
// raise (runtime.py:335-343); the CTA leaves its block loop at the next
// block boundary (__syncthreads_or of the flags)
__device__ __forceinline__ void bf_trap(const BfJitGeom& G, int kind, long long blk, bool& t) {
  t = true;
  if (atomicCAS(G.fault, 0, kind) == 0) {
    *reinterpret_cast<long long*>(G.fault + 2) = blk;
    *reinterpret_cast<unsigned long long*>(G.fault + 4) = G.task;
    __threadfence_system();
    int* hf = *reinterpret_cast<int* const*>(G.fault + 6);
    if (hf) *(volatile int*)hf = 1;
  }
}
__device__ __forceinline__ int bf_add32(int a, int b) { return (int)((unsigned)a + (unsigned)b); }
__device__ __forceinline__ int bf_sub32(int a, int b) { return (int)((unsigned)a - (unsigned)b); }
__device__ __forceinline__ int bf_mul32(int a, int b) { return (int)((unsigned)a * (unsigned)b); }
__device__ __forceinline__ int bf_neg32(int a) { return (int)(0u - (unsigned)a); }
__device__ __forceinline__ long long bf_add64(long long a, long long b) { return (long long)((unsigned long long)a + (unsigned long long)b); }
__device__ __forceinline__ long long bf_sub64(long long a, long long b) { return (long long)((unsigned long long)a - (unsigned long long)b); }
__device__ __forceinline__ long long bf_mul64(long long a, long long b) { return (long long)((unsigned long long)a * (unsigned long long)b); }
__device__ __forceinline__ long long bf_neg64(long long a) { return (long long)(0ull - (unsigned long long)a); }
"""

HELPERS = r"""
#define BF_DIV_INT(T, NEG)                                                        \
  __device__ __forceinline__ T bf_div_##T(T a, T b, const BfJitGeom& G, long long blk, bool& t) { \
    if (b == 0) { bf_trap(G, 2, blk, t); return 0; }                                 \
    if (b == -1) return NEG(a);                                                   \
    return a / b;                                                                 \
  }                                                                               \
  __device__ __forceinline__ T bf_mod_##T(T a, T b, const BfJitGeom& G, long long blk, bool& t) { \
    if (b == 0) { bf_trap(G, 2, blk, t); return 0; }                                 \
    if (b == -1) return 0;                                                        \
    return a % b;                                                                 \
  }
typedef long long ll;
BF_DIV_INT(int, bf_neg32)
BF_DIV_INT(ll, bf_neg64)
__device__ __forceinline__ double bf_fdiv(double a, double b, const BfJitGeom& G, long long blk, bool& t) {
  if (b == 0.0) { bf_trap(G, 2, blk, t); return 0.0; }
  return a / b;
}
__device__ __forceinline__ double bf_sqrt(double a, const BfJitGeom& G, long long blk, bool& t) {
  if (a < 0.0) { bf_trap(G, 3, blk, t); return 0.0; }
  return sqrt(a);
}
__device__ __forceinline__ int bf_abs32(int a) { return a < 0 ? bf_neg32(a) : a; }
__device__ __forceinline__ ll bf_abs64(ll a) { return a < 0 ? bf_neg64(a) : a; }
// f32 atomic add with the reference's rounding: new = RN32(old + operand)
__device__ __forceinline__ void bf_atomic_add_f32(float* p, double v) {
  unsigned* u = reinterpret_cast<unsigned*>(p);
  unsigned old = *u, assumed;
  do {
    assumed = old;
    const float nv = (float)((double)__uint_as_float(assumed) + v);
    old = atomicCAS(u, assumed, __float_as_uint(nv));
  } while (old != assumed);
}
__device__ __forceinline__ void bf_atomic_cas_f32(float* p, double cmp, double v) {
  unsigned* u = reinterpret_cast<unsigned*>(p);
  unsigned old = *u;
  while ((double)__uint_as_float(old) == cmp) {
    const unsigned got = atomicCAS(u, old, __float_as_uint((float)v));
    if (got == old) return;
    old = got;
  }
}
__device__ __forceinline__ void bf_atomic_cas_f64(double* p, double cmp, double v) {
  unsigned long long* u = reinterpret_cast<unsigned long long*>(p);
  unsigned long long old = *u;
  while (__longlong_as_double((long long)old) == cmp) {
    const unsigned long long got = atomicCAS(u, old, (unsigned long long)__double_as_longlong(v));
    if (got == old) return;
    old = got;
  }
}
"""


class _Gen:
    def __init__(self, mk):
        self.mk = mk
        self.params = list(mk.param_signature)
        self.local_types = dict(getattr(mk, "local_types", {}))
        self.memory_map = dict(getattr(mk, "memory_map", {}))
        self.layout = mk.shared_layout
        self.warp_mode = bool(getattr(mk, "warp_mode", False))
        self.tmp = 0
        self.uses_xchg = False
        self.scalars = {}   # name -> dsl type (params)
        self.arrays = {}    # name -> (space, dsl type, c ptr expr, c len expr)
        for i, p in enumerate(self.params):
            if p.ptype.is_global:
                self.arrays[p.name] = ("global", p.ptype.scalar, f"p_{p.name}", f"n_{p.name}")
            else:
                self.scalars[p.name] = p.ptype.scalar
        for slot, d in enumerate(self.layout.static):
            self.arrays[d.name] = ("shared", d.scalar, f"s_{d.name}", str(d.length))
        for name, ref in self.memory_map.items():
            if ref.space == "shared-dynamic":
                self.arrays[name] = ("dyn", self.layout.dynamic_scalar, f"d_{name}", "G.dyn_elems")

    # -- types ---------------------------------------------------------------
    def var_type(self, name: str) -> str:
        if name in self.local_types:
            return self.local_types[name]
        if name in self.scalars:
            return self.scalars[name]
        raise CodegenError(f"unknown variable {name!r}")

    def new_tmp(self) -> str:
        self.tmp += 1
        return f"_t{self.tmp}"

    # -- expressions ---------------------------------------------------------
    def expr(self, e, out: list, subst: dict) -> tuple[str, str]:
        """-> (C expression, DSL type).  `out` receives hoisted statements."""
        k = _cls(e)
        if k == "IntLit":
            ty = e.ty or "i32"
            if ty in ("f32", "f64"):
                return _float_lit(float(e.value)), ty
            if ty == "i64":
                v = (int(e.value) + 2**63) % 2**64 - 2**63
                return f"({v}LL)", ty
            v = (int(e.value) + 2**31) % 2**32 - 2**31
            return (f"({v})" if v != -2**31 else "(-2147483647-1)"), "i32"
        if k == "FloatLit":
            return _float_lit(float(e.value)), e.ty or "f64"
        if k == "VarRef":
            if id(e) in subst:
                return subst[id(e)]
            return f"v_{e.name}", self.var_type(e.name)
        if k == "BuiltinRef":
            return f"{e.base}_{e.axis}", "i32"
        if k == "Index":
            space, ety, ptr, ln = self.arrays[e.array]
            idx, ity = self.expr(e.index, out, subst)
            t = self.new_tmp()
            out.append(f"long long {t}_i = (long long)({idx});")
            out.append(f"{_CTYPE[ety]} {t} = 0;")
            out.append(f"if ({t}_i < 0 || {t}_i >= (long long)({ln})) bf_trap(G, 1, blk, bf_t); "
                       f"else {t} = ({_CTYPE[ety]}){ptr}[{t}_i];")
            return t, ety
        if k == "Binary":
            return self.binary(e, out, subst)
        if k == "Unary":
            v, ty = self.expr(e.operand, out, subst)
            if e.op == "!":
                return f"(({v}) == 0 ? 1 : 0)", "i32"
            ty = e.ty or ty
            if ty == "i32":
                return f"bf_neg32({v})", ty
            if ty == "i64":
                return f"bf_neg64({v})", ty
            return f"(-({v}))", ty
        if k == "Call":
            if id(e) in subst:
                return subst[id(e)]
            if e.func in WARP_INTRINSICS:
                raise CodegenError("warp intrinsic outside a lockstep statement")
            args = [self.expr(a, out, subst) for a in e.args]
            ty = e.ty or args[0][1]
            if e.func in ("min", "max"):
                a, b = args[0][0], args[1][0]
                ta, tb = self.new_tmp(), self.new_tmp()
                out.append(f"{_CTYPE[ty]} {ta} = {a}; {_CTYPE[ty]} {tb} = {b};")
                # Python min/max: min(a, b) is a unless b < a
                return (f"(({tb} < {ta}) ? {tb} : {ta})" if e.func == "min"
                        else f"(({tb} > {ta}) ? {tb} : {ta})"), ty
            if e.func == "abs":
                a = args[0][0]
                if ty == "i32":
                    return f"bf_abs32({a})", ty
                if ty == "i64":
                    return f"bf_abs64({a})", ty
                return f"fabs({a})", ty
            if e.func == "sqrt":
                return f"bf_sqrt((double)({args[0][0]}), G, blk, bf_t)", ty if ty in ("f32", "f64") else "f64"
            raise CodegenError(f"unknown intrinsic {e.func!r}")
        raise CodegenError(f"unknown expression node {k}")

    def binary(self, e, out, subst):
        op = e.op
        if op in ("&&", "||"):
            # short-circuit: the right side's hoisted loads must stay conditional
            lv, _ = self.expr(e.left, out, subst)
            t = self.new_tmp()
            out.append(f"int {t} = ({lv}) != 0 ? 1 : 0;")
            rout: list = []
            rv, _ = self.expr(e.right, rout, subst)
            cond = f"{t}" if op == "&&" else f"!{t}"
            out.append(f"if ({cond}) {{ " + " ".join(rout) + f" {t} = ({rv}) != 0 ? 1 : 0; }}")
            return t, "i32"
        lv, lt = self.expr(e.left, out, subst)
        rv, rt = self.expr(e.right, out, subst)
        if op in ("==", "!=", "<", "<=", ">", ">="):
            return f"(({lv}) {op} ({rv}) ? 1 : 0)", "i32"
        ty = e.ty or lt
        if ty in ("i32", "i64"):
            w = "32" if ty == "i32" else "64"
            c = "int" if ty == "i32" else "ll"
            if op == "+":
                return f"bf_add{w}({lv}, {rv})", ty
            if op == "-":
                return f"bf_sub{w}({lv}, {rv})", ty
            if op == "*":
                return f"bf_mul{w}({lv}, {rv})", ty
            if op == "/":
                return f"bf_div_{c}({lv}, {rv}, G, blk, bf_t)", ty
            if op == "%":
                return f"bf_mod_{c}({lv}, {rv}, G, blk, bf_t)", ty
        else:
            if op in ("+", "-", "*"):
                return f"((double)({lv}) {op} (double)({rv}))", ty
            if op == "/":
                return f"bf_fdiv((double)({lv}), (double)({rv}), G, blk, bf_t)", ty
            if op == "%":
                out.append("bf_trap(G, 3, blk, bf_t);")
                return "0.0", ty
        raise CodegenError(f"unknown operator {op!r}")

    def coerce(self, v: str, src: str, dst: str) -> str:
        if dst in ("i32", "i64"):
            c = _CTYPE[dst]
            if src in ("f32", "f64"):
                return f"({c})(long long)({v})"
            if dst == "i32" and src == "i64":
                return f"(int)(unsigned)(unsigned long long)({v})"
            return f"({c})({v})"
        return f"(double)({v})"

    # -- statements ----------------------------------------------------------
    def warp_calls(self, e, acc: list) -> None:
        k = _cls(e)
        if k == "Call":
            for a in e.args:
                self.warp_calls(a, acc)
            if e.func in WARP_INTRINSICS:
                acc.append(e)
        elif k == "Binary":
            self.warp_calls(e.left, acc)
            self.warp_calls(e.right, acc)
        elif k == "Unary":
            self.warp_calls(e.operand, acc)
        elif k == "Index":
            self.warp_calls(e.index, acc)

    def stmt_exprs(self, s) -> list:
        k = _cls(s)
        if k == "LocalDecl":
            return [s.init]
        if k == "Assign":
            return [s.value] + ([s.target.index] if s.target.index is not None else [])
        if k == "AtomicStmt":
            return [s.operand] + ([s.target.index] if s.target.index is not None else []) + \
                   ([s.compare_to] if s.compare_to is not None else [])
        return []

    def lockstep(self, s, lines: list, subst: dict, ind: str) -> dict:
        """Hoist the warp intrinsics of statement s (post-order) through the
        shared exchange buffer; returns the substitution for the statement."""
        calls: list = []
        for ex in self.stmt_exprs(s):
            self.warp_calls(ex, calls)
        subst = dict(subst)
        for call in calls:
            self.uses_xchg = True
            out: list = []
            if call.func == "shfl_down":
                v, ty = self.expr(call.args[0], out, subst)
                d, _ = self.expr(call.args[1], out, subst)
                r = self.new_tmp()
                lines.extend(ind + x for x in out)
                lines.append(f"{ind}__syncthreads();")
                if ty in ("f32", "f64"):
                    lines.append(f"{ind}xchg_d[tid] = (double)({v});")
                else:
                    lines.append(f"{ind}xchg_l[tid] = (long long)({v});")
                lines.append(f"{ind}__syncthreads();")
                lines.append(f"{ind}{_CTYPE[ty]} {r};")
                lines.append(f"{ind}{{ long long src = (long long)wlane + (long long)({d});"
                             f" if (src >= 0 && src < wlim) {r} = ({_CTYPE[ty]})"
                             f"{'xchg_d' if ty in ('f32', 'f64') else 'xchg_l'}[wbase + src];"
                             f" else {r} = ({_CTYPE[ty]})"
                             f"{'xchg_d' if ty in ('f32', 'f64') else 'xchg_l'}[tid]; }}")
                subst[id(call)] = (r, ty)
            else:
                p, _ = self.expr(call.args[0], out, subst)
                r = self.new_tmp()
                lines.extend(ind + x for x in out)
                lines.append(f"{ind}__syncthreads();")
                lines.append(f"{ind}xchg_l[tid] = (({p}) != 0) ? 1 : 0;")
                lines.append(f"{ind}__syncthreads();")
                if call.func == "vote_any":
                    lines.append(f"{ind}int {r} = 0; for (int q = 0; q < wcount; q++) "
                                 f"if (xchg_l[wbase + q]) {{ {r} = 1; break; }}")
                else:
                    lines.append(f"{ind}int {r} = 1; for (int q = 0; q < wcount; q++) "
                                 f"if (!xchg_l[wbase + q]) {{ {r} = 0; break; }}")
                subst[id(call)] = (r, "i32")
        return subst

    def has_warp(self, s) -> bool:
        calls: list = []
        for ex in self.stmt_exprs(s):
            self.warp_calls(ex, calls)
        if calls:
            return True
        k = _cls(s)
        if k == "For":
            return any(self.has_warp(x) for x in s.body)
        if k == "If":
            return any(self.has_warp(x) for x in s.then_body + s.else_body)
        return False

    def stmts(self, body, lines: list, ind: str, in_if: bool = False) -> None:
        for s in body:
            self.stmt(s, lines, ind, in_if)

    def stmt(self, s, lines: list, ind: str, in_if: bool) -> None:
        k = _cls(s)
        subst: dict = {}
        if self.warp_mode and k in ("LocalDecl", "Assign", "AtomicStmt") and self.has_warp(s):
            if in_if:  # interp.py:325-327
                lines.append(f"{ind}bf_trap(G, 4, blk, bf_t);")
                return
            subst = self.lockstep(s, lines, subst, ind)
        out: list = []
        if k == "LocalDecl":
            v, ty = self.expr(s.init, out, subst)
            lines.extend(ind + x for x in out)
            lines.append(f"{ind}v_{s.name} = {self.coerce(v, ty, s.ty)};")
        elif k == "Assign":
            if s.target.index is None:
                v, ty = self.expr(s.value, out, subst)
                dst = self.var_type(s.target.name)
                lines.extend(ind + x for x in out)
                lines.append(f"{ind}v_{s.target.name} = {self.coerce(v, ty, dst)};")
            else:
                # value first, then index (exec_stmt, interp.py:159-165)
                v, ty = self.expr(s.value, out, subst)
                space, ety, ptr, ln = self.arrays[s.target.name]
                idx, _ = self.expr(s.target.index, out, subst)
                lines.extend(ind + x for x in out)
                t = self.new_tmp()
                lines.append(f"{ind}{{ long long {t} = (long long)({idx}); "
                             f"if ({t} < 0 || {t} >= (long long)({ln})) bf_trap(G, 1, blk, bf_t); "
                             f"else {ptr}[{t}] = ({_MTYPE[ety]})({self.coerce(v, ty, ety)}); }}")
        elif k == "If":
            c, _ = self.expr(s.cond, out, subst)
            lines.extend(ind + x for x in out)
            lines.append(f"{ind}if (({c}) != 0) {{")
            self.stmts(s.then_body, lines, ind + "  ", True)
            if s.else_body:
                lines.append(f"{ind}}} else {{")
                self.stmts(s.else_body, lines, ind + "  ", True)
            lines.append(f"{ind}}}")
        elif k == "For":
            lo, lty = self.expr(s.lo, out, subst)
            lines.extend(ind + x for x in out)
            lines.append(f"{ind}v_{s.var} = {self.coerce(lo, lty, 'i32')};")
            lines.append(f"{ind}for (;;) {{")
            hout: list = []
            hi, hty = self.expr(s.hi, hout, {})
            lines.extend(ind + "  " + x for x in hout)
            lines.append(f"{ind}  if (!(v_{s.var} < ({hi})) || bf_t) break;")
            self.stmts(s.body, lines, ind + "  ", in_if)
            sout: list = []
            st, sty = self.expr(s.step, sout, {})
            lines.extend(ind + "  " + x for x in sout)
            lines.append(f"{ind}  v_{s.var} = bf_add32(v_{s.var}, {self.coerce(st, sty, 'i32')});")
            lines.append(f"{ind}}}")
        elif k == "AtomicStmt":
            space, ety, ptr, ln = self.arrays[s.target.name]
            if s.target.index is None:
                lines.append(f"{ind}bf_trap(G, 3, blk, bf_t);")
                return
            idx, _ = self.expr(s.target.index, out, subst)
            opv, oty = self.expr(s.operand, out, subst)
            cmp = None
            if s.compare_to is not None:
                cmp, cty = self.expr(s.compare_to, out, subst)
            lines.extend(ind + x for x in out)
            t = self.new_tmp()
            lines.append(f"{ind}{{ long long {t} = (long long)({idx});")
            lines.append(f"{ind}  if ({t} < 0 || {t} >= (long long)({ln})) bf_trap(G, 1, blk, bf_t); else if (!bf_t) {{")
            a = f"&{ptr}[{t}]"
            if s.kind == "add":
                if ety == "i32":
                    lines.append(f"{ind}    atomicAdd((unsigned*){a}, (unsigned)({self.coerce(opv, oty, 'i32')}));")
                elif ety == "i64":
                    lines.append(f"{ind}    atomicAdd((unsigned long long*){a}, (unsigned long long)({self.coerce(opv, oty, 'i64')}));")
                elif ety == "f32":
                    lines.append(f"{ind}    bf_atomic_add_f32({a}, (double)({opv}));")
                else:
                    lines.append(f"{ind}    atomicAdd({a}, (double)({opv}));")
            else:
                if ety == "i32":
                    lines.append(f"{ind}    atomicCAS((unsigned*){a}, (unsigned)({self.coerce(cmp, cty, 'i32')}), "
                                 f"(unsigned)({self.coerce(opv, oty, 'i32')}));")
                elif ety == "i64":
                    lines.append(f"{ind}    atomicCAS((unsigned long long*){a}, (unsigned long long)"
                                 f"({self.coerce(cmp, cty, 'i64')}), (unsigned long long)({self.coerce(opv, oty, 'i64')}));")
                elif ety == "f32":
                    lines.append(f"{ind}    bf_atomic_cas_f32({a}, (double)({cmp}), (double)({opv}));")
                else:
                    lines.append(f"{ind}    bf_atomic_cas_f64({a}, (double)({cmp}), (double)({opv}));")
            lines.append(f"{ind}  }} }}")
        elif k in ("Noop",):
            pass
        elif k == "Barrier":
            lines.append(f"{ind}__syncthreads();")
        else:
            raise CodegenError(f"unknown statement node {k}")

    # -- kernel --------------------------------------------------------------
    def kernel(self, entry: str) -> str:
        nw = max(2 * len(self.params), 2)
        body: list = []
        ind = "    "
        for si, sec in enumerate(self.mk.sections):
            if _cls(sec) == "ThreadSection":
                self.stmts(sec.body, body, ind)
            else:  # LoopSection: uniform loop, phases separated by barriers
                out: list = []
                lo, lty = self.expr(sec.lo, out, {})
                body.extend(ind + x for x in out)
                body.append(f"{ind}v_{sec.var} = {self.coerce(lo, lty, 'i32')};")
                body.append(f"{ind}for (;;) {{")
                hout: list = []
                hi, _ = self.expr(sec.hi, hout, {})
                body.extend(ind + "  " + x for x in hout)
                body.append(f"{ind}  if (!(v_{sec.var} < ({hi}))) break;")
                for pi, phase in enumerate(sec.phases):
                    if pi > 0:
                        body.append(f"{ind}  __syncthreads();")
                    self.stmts(phase, body, ind + "  ")
                sout: list = []
                st, sty = self.expr(sec.step, sout, {})
                body.extend(ind + "  " + x for x in sout)
                body.append(f"{ind}  v_{sec.var} = bf_add32(v_{sec.var}, {self.coerce(st, sty, 'i32')});")
                body.append(f"{ind}  if (__syncthreads_or(bf_t)) break;")
                body.append(f"{ind}}}")
            if si in getattr(self.mk, "barrier_boundaries", set()):
                body.append(f"{ind}__syncthreads();")

        src = [PRELUDE % {"nw": nw}, HELPERS]
        src.append(f'extern "C" __global__ void __launch_bounds__(1024) {entry}(const BfJitArgs A, const BfJitGeom G) {{')
        # parameters
        for i, p in enumerate(self.params):
            if p.ptype.is_global:
                src.append(f"  {_MTYPE[p.ptype.scalar]}* p_{p.name} = "
                           f"reinterpret_cast<{_MTYPE[p.ptype.scalar]}*>(A.w[{2 * i}]);")
                src.append(f"  const long long n_{p.name} = A.w[{2 * i + 1}];")
            else:
                sc = p.ptype.scalar
                if sc in ("f32", "f64"):
                    src.append(f"  const double v_{p.name} = __longlong_as_double(A.w[{2 * i}]);")
                elif sc == "i64":
                    src.append(f"  const long long v_{p.name} = A.w[{2 * i}];")
                else:
                    src.append(f"  const int v_{p.name} = (int)A.w[{2 * i}];")
        for d in self.layout.static:
            src.append(f"  __shared__ {_MTYPE[d.scalar]} s_{d.name}[{d.length}];")
        dyn_names = [n for n, (sp, *_r) in self.arrays.items() if sp == "dyn"]
        if dyn_names:
            dt = _MTYPE[self.layout.dynamic_scalar]
            src.append(f"  extern __shared__ __align__(16) unsigned char bf_dyn[];")
            for n in dyn_names:
                src.append(f"  {dt}* d_{n} = reinterpret_cast<{dt}*>(bf_dyn);")
        if self.uses_xchg:
            src.append("  __shared__ long long xchg_l[1024];")
            src.append("  __shared__ double xchg_d[1024];")
        for name, ty in self.local_types.items():
            src.append(f"  {_CTYPE[ty]} v_{name} = 0;")
        src.append("  const int tid = threadIdx.x;")
        src.append("  const int B = G.bx * G.by * G.bz;")
        src.append("  const int threadIdx_x = tid % G.bx, threadIdx_y = (tid / G.bx) % G.by, "
                   "threadIdx_z = tid / (G.bx * G.by);")
        src.append("  const int blockDim_x = G.bx, blockDim_y = G.by, blockDim_z = G.bz;")
        src.append("  const int gridDim_x = G.gx, gridDim_y = G.gy, gridDim_z = G.gz;")
        src.append("  const int ws = G.warp_size > 0 ? G.warp_size : 32;")
        src.append("  const int wbase = (tid / ws) * ws, wlane = tid - wbase;")
        src.append("  const int wcount = (B - wbase) < ws ? (B - wbase) : ws;")
        src.append("  const long long wlim = wcount;")
        src.append("  (void)wlane; (void)wlim; (void)B;")
        src.append("  bool bf_t = false;  // this thread trapped")
        # static mode: one pass of the grid over [first, first + count); device
        # fetching: claims of `grain` blocks until the task is drained (a trap
        # abandons the rest of its fetch only, runtime.py:335-343)
        src.append("  const bool bf_dev = G.dcur != nullptr;")
        src.append("  int bf_sub = (int)(blockIdx.x % 8), bf_tried = 0;")
        src.append("  unsigned long long bf_nclaims = 0, bf_nblocks = 0;")
        src.append("  long long bf_f = bf_dev ? bf_take(tid == 0 ? bf_claim(G, bf_sub, bf_tried, bf_nclaims) : 0) : 0;")
        src.append("  const long long bf_nf = bf_dev ? G.nfetch : 1;")
        src.append("  while (bf_f < bf_nf) {")
        src.append("  const long long bf_nx = bf_dev && tid == 0 ? bf_claim(G, bf_sub, bf_tried, bf_nclaims) : 0;")
        src.append("  const long long bf_b0 = bf_dev ? G.first + bf_f * G.grain : G.first;")
        src.append("  const long long bf_b1 = bf_dev ? (bf_b0 + G.grain < G.first + G.count ? bf_b0 + G.grain "
                   ": G.first + G.count) : G.first + G.count;")
        src.append("  bf_t = false;")
        src.append("  for (long long blk = bf_b0 + (bf_dev ? 0 : blockIdx.x); blk < bf_b1; "
                   "blk += (bf_dev ? 1 : gridDim.x)) {")
        src.append("    const int blockIdx_x = (int)(blk % G.gx), blockIdx_y = (int)((blk / G.gx) % G.gy), "
                   "blockIdx_z = (int)(blk / ((long long)G.gx * G.gy));")
        src.append("    (void)blockIdx_x; (void)blockIdx_y; (void)blockIdx_z;")
        for d in self.layout.static:
            src.append(f"    for (int i = tid; i < {d.length}; i += B) s_{d.name}[i] = 0;")
        for n in dyn_names:
            src.append(f"    for (long long i = tid; i < G.dyn_elems; i += B) d_{n}[i] = 0;")
            break
        for name, ty in self.local_types.items():
            src.append(f"    v_{name} = 0;")
        src.append("    __syncthreads();")
        src.extend(body)
        src.append("    if (__syncthreads_or(bf_t)) break;")
        src.append("    if (bf_dev && tid == 0) {")
        src.append("      bf_nblocks++;")
        src.append("      if (G.dexec) atomicAdd(G.dexec + blk, 1);")
        src.append("    }")
        src.append("  }")
        src.append("  if (!bf_dev) break;")
        src.append("  bf_f = bf_take(bf_nx);")
        src.append("  }")
        src.append("  if (bf_dev && tid == 0 && bf_nclaims) {")
        src.append("    atomicAdd(G.dstats + 2 * (blockIdx.x % G.dslots), bf_nclaims);")
        src.append("    atomicAdd(G.dstats + 2 * (blockIdx.x % G.dslots) + 1, bf_nblocks);")
        src.append("  }")
        src.append("}")
        return "\n".join(src) + "\n"


def fingerprint(mk) -> str:
    d = mk.to_dict()
    import json
    return hashlib.sha256(json.dumps(d, sort_keys=True).encode()).hexdigest()


def generate(mk) -> tuple[str, str, list]:
    """-> (CUDA source, entry name, param spec [(slot kind, scalar)])."""
    fp = fingerprint(mk)
    entry = f"bfjit_{fp[:16]}"
    src = _Gen(mk).kernel(entry)
    spec = []
    for p in mk.param_signature:
        if p.ptype.is_global:
            spec.append(("handle", p.ptype.scalar))
        else:
            spec.append((p.ptype.scalar, None))
    return src, entry, spec
