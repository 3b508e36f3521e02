// Run-time specialised fused-pass kernels (the K5 pass without an interpreter).
//
// The ahead-of-time kernel k_fused walks an op table in shared memory and
// dispatches every run of ops through a switch over ~70 template bodies; the
// dispatch (a compare tree plus an indirect branch, taken by every warp for
// every op of every tile) costs several hundred cycles per op, more than the
// op's arithmetic.  A pass's op sequence is identical for all 2^(n-K) tiles,
// so this file turns the planned pass (FParams: stages, lowered ops) into a
// straight-line program — every op a call of pair_ct / phase_ct with its
// slot, class, register mask and gate entries as compile-time constants and
// its thread / tile predicate as a literal mask test — compiles it with NVRTC
// for sm_100a, and launches it with the same kernel body (fused_body), grid,
// ring and register layouts as k_fused.  Same layouts, same per-pair
// arithmetic, same `one` opaque to ptxas: the results are the interpreter's
// bit for bit (tests run every fused case both ways).
//
// Policy (QSB_FUSED_JIT): 0 = off; 1 (default) = queue the compile on the
// first launch of a pass and keep interpreting it until the program is ready
// (NVRTC runs on host worker threads, nothing blocks); 2 = compile
// synchronously and always launch the program.  qs_jit_sync waits for the
// queued compiles (benchmarks call it after warm-up).  Compiled programs are
// cached per device for the life of the process.  NVRTC is loaded with
// dlopen; without it the interpreter kernel runs (same device code path, no
// CPU fallback).

#include <dlfcn.h>
#include <sys/stat.h>
#include <pthread.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <set>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "fused_dev.cuh"
#include "internal.h"

namespace qsb {

namespace {

#include "_jit_headers.inc"  // kJitCommon, kJitFusedDev: the two headers as text (build.py)

// ---- NVRTC, loaded lazily ---------------------------------------------------
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram *nvrtcProgram_t;
struct Nvrtc {
    bool ok = false;
    nvrtcResult_t (*create)(nvrtcProgram_t *, const char *, const char *, int, const char *const *,
                            const char *const *);
    nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char *const *);
    nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t *);
    nvrtcResult_t (*log)(nvrtcProgram_t, char *);
    nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t *);
    nvrtcResult_t (*cubin)(nvrtcProgram_t, char *);
    nvrtcResult_t (*destroy)(nvrtcProgram_t *);
    int major = 0, minor = 0;
};

Nvrtc load_nvrtc() {
    Nvrtc n;
    // The toolkit's NVRTC by absolute path first: a bare "libnvrtc.so.12"
    // resolves to whichever copy the process already holds — under torch its
    // bundled (older) one, whose ptxas builds every packed FFMA2 multiplier as
    // a register pair (two MOVs each; the H-layer's first pass 2.63 -> 3.1 ms).
    // QSB_NVRTC overrides.
    const char *names[] = {std::getenv("QSB_NVRTC"), "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12",
                           "libnvrtc.so"};
    void *h = nullptr;
    for (const char *nm : names)
        if (nm && *nm && (h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return n;
    if (auto ver = (nvrtcResult_t(*)(int *, int *))dlsym(h, "nvrtcVersion")) ver(&n.major, &n.minor);
    n.create = (decltype(n.create))dlsym(h, "nvrtcCreateProgram");
    n.compile = (decltype(n.compile))dlsym(h, "nvrtcCompileProgram");
    n.log_size = (decltype(n.log_size))dlsym(h, "nvrtcGetProgramLogSize");
    n.log = (decltype(n.log))dlsym(h, "nvrtcGetProgramLog");
    n.cubin_size = (decltype(n.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
    n.cubin = (decltype(n.cubin))dlsym(h, "nvrtcGetCUBIN");
    n.destroy = (decltype(n.destroy))dlsym(h, "nvrtcDestroyProgram");
    n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy;
    return n;
}

// loaded once, thread-safe (function-local static initialisation)
const Nvrtc &nvrtc() {
    static const Nvrtc n = load_nvrtc();
    return n;
}

// ---- driver entry points ------------------------------------------------------
struct Driver {
    bool ok = false;
    PFN_cuModuleLoadData_v2000 load;
    PFN_cuModuleGetFunction_v2000 get;
    PFN_cuFuncSetAttribute_v9000 set_attr;
    PFN_cuLaunchKernel_v4000 launch;
};

Driver load_driver() {
    Driver d;
    auto sym = [](const char *name) -> void * {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return fn;
    };
    d.load = (PFN_cuModuleLoadData_v2000)sym("cuModuleLoadData");
    d.get = (PFN_cuModuleGetFunction_v2000)sym("cuModuleGetFunction");
    d.set_attr = (PFN_cuFuncSetAttribute_v9000)sym("cuFuncSetAttribute");
    d.launch = (PFN_cuLaunchKernel_v4000)sym("cuLaunchKernel");
    d.ok = d.load && d.get && d.set_attr && d.launch;
    return d;
}

const Driver &driver() {
    static const Driver d = load_driver();
    return d;
}

// ---- code generation -----------------------------------------------------------
// Runs of one variant at least kJitLoopRun long (each op touching at least
// kJitLoopMinRegs float4 registers) may stay loops over the shared-memory op
// table instead of straight-line code (smaller programs).  Measured on B200
// the straight-line form is faster even when the program overflows the
// instruction cache (QFT(28) 8.26 -> 8.14 ms, QFT(30) 35.3 -> 34.8 ms,
// config 4 1002 -> 977 ms; 150 tile-tested phases 4.6 -> 4.1 ms), so loops
// are off by default; QSB_JIT_LOOP_RUN=<n> turns them back on.
constexpr int kJitLoopRun = 1 << 30;
constexpr int kJitLoopMinRegs = 8;
void hexf(std::string &out, float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    char buf[40];
    std::snprintf(buf, sizeof buf, "__int_as_float(0x%08x)", b);
    out += buf;
}

// An op's thread / tile predicate as generated source: the uniform tests
// (tile bits against the redux'd base `ub`, warp bits against `wid`) and the
// divergent lane test; "" when the op applies everywhere.
std::string uniform_test(const FOp &op) {
    std::string test;
    char buf[96];
    if (op.ext_need) {
        std::snprintf(buf, sizeof buf, "(ub & 0x%llxull) == 0x%llxull", (unsigned long long)op.ext_need,
                      (unsigned long long)op.ext_need);
        test += buf;
    }
    if (op.tid_need & ~31u) {
        std::snprintf(buf, sizeof buf, "(wid & 0x%xu) == 0x%xu", op.tid_need & ~31u, op.tid_need & ~31u);
        if (!test.empty()) test += " && ";
        test += buf;
    }
    return test;
}

std::string lane_test(const FOp &op) {
    if (!(op.tid_need & 31u)) return "";
    char buf[64];
    std::snprintf(buf, sizeof buf, "(tid & 0x%xu) == 0x%xu", op.tid_need & 31u, op.tid_need & 31u);
    return buf;
}

std::string op_test(const FOp &op) {
    std::string u = uniform_test(op), l = lane_test(op);
    if (u.empty()) return l;
    if (l.empty()) return u;
    return u + " && " + l;
}

// A unit-modulus diagonal entry d = e^{i theta} as fixed-point turns
// (theta / 2 pi * 2^32, modulo 2^32); false when |d| is not 1.
bool unit_turns(const FOp &op, uint32_t *turns) {
    const double x = op.m[6], y = op.m[7];
    if (std::fabs(std::sqrt(x * x + y * y) - 1.0) > 1e-6) return false;
    double t = std::atan2(y, x) / (2.0 * 3.14159265358979323846);
    if (t < 0) t += 1.0;
    *turns = (uint32_t)(uint64_t)std::llround(t * 4294967296.0);
    return true;
}

// QSB_JIT_STATIC_STAGES=0: generated programs use fused_body's generic
// stage loop (layouts from the parameter block), for measurements
bool static_stages_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("QSB_JIT_STATIC_STAGES");
        return !(e && e[0] == '0');
    }();
    return on;
}

// The whole stage sequence of a generated program with the stage layouts as
// literals: each thread's padded shared-memory base per stage is a few
// shifts of its lane / warp bits (loop-invariant across tiles) and every
// register's offset the immediate of a 128-bit ld/st.shared.  The generic
// loop in fused_body reads the layouts from the parameter block and
// rebuilds the addresses per stage and tile (about as many instructions as
// the ops of a light pass).  dbl: complex128 registers (one amplitude per
// 16-B unit).
void emit_run_stages(std::string &src, const FParams &p, int RB, bool dbl) {
    char buf[256];
    const char *vt = dbl ? "double2" : "float4";
    src += "  static constexpr bool kOwnsStages = true;\n"
           "  template <int RB_, int NC>\n"
           "  static __device__ __forceinline__ void run_stages(float4 *tile, uint32_t tid, uint64_t base,\n"
           "      float one, const FOp *ops) {\n"
           "    const uint32_t lane = tid & 31u, warp = tid >> 5;\n    (void)warp;\n    const FStage st0{};\n";
    for (int k = 0; k < p.nstages; ++k) {
        const FStage &st = p.stages[k];
        std::string fb = "0u";
        for (int q = 0; q < 5; ++q) {
            std::snprintf(buf, sizeof buf, " | (((lane >> %d) & 1u) << %d)", q, st.lf[q]);
            fb += buf;
        }
        for (int q = 0; q < p.nwbits; ++q) {
            std::snprintf(buf, sizeof buf, " | (((warp >> %d) & 1u) << %d)", q, st.wf[q]);
            fb += buf;
        }
        src += "    { // stage " + std::to_string(k) + "\n      const uint32_t fb = " + fb +
               ";\n      const uint32_t sb = smem_u32(tile) + (fb + (fb >> 5)) * 16u;\n      " + vt +
               " v[1 << RB_];\n";
        std::vector<uint32_t> off(1u << RB);
        for (int j = 0; j < (1 << RB); ++j) {
            uint32_t a = 0;
            for (int r = 0; r < RB; ++r)
                if (j & (1 << r)) a += (1u << st.rf[r]) + ((1u << st.rf[r]) >> 5);
            off[j] = a;
        }
        for (int j = 0; j < (1 << RB); ++j) {
            std::snprintf(buf, sizeof buf, "      v[%d] = %s(sb + %uu);\n", j, dbl ? "lds128d" : "lds128", 16u * off[j]);
            src += buf;
        }
        std::snprintf(buf, sizeof buf, "      run<RB_>(%d, st0, ops, tid, base, one, v);\n", k);
        src += buf;
        for (int j = 0; j < (1 << RB); ++j) {
            std::snprintf(buf, sizeof buf, "      %s(sb + %uu, v[%d]);\n", dbl ? "sts128d" : "sts128", 16u * off[j], j);
            src += buf;
        }
        if (k + 1 < p.nstages) src += "      named_sync(1, NC);\n";
        src += "    }\n";
    }
    src += "  }\n";
}

std::string generate(const FParams &p, int K, int RB, bool param = false) {
    // diagonal ops inside a test: 0 (default) packed phase_ct, 1 scalar
    // phase_cs, 2 scalar everywhere (QSB_JIT_PHASE, for measurements).  The
    // scalar in-branch form won under the older NVRTC, whose packed results
    // needed copies home after a branch; with the toolkit's NVRTC the packed
    // form is faster (QFT(30) 28.4 -> 27.9 ms)
    int phase_mode = 0;
    if (const char *e = std::getenv("QSB_JIT_PHASE")) phase_mode = std::atoi(e);
    int loop_run = kJitLoopRun;
    if (const char *e = std::getenv("QSB_JIT_LOOP_RUN")) loop_run = std::atoi(e);
    // ops under a LANE test: 1 (default) predicated selection (phase_sel /
    // swap_sel: no divergent branch), 0 a branch around the body
    int sel_mode = 1;
    if (const char *e = std::getenv("QSB_JIT_SEL")) sel_mode = std::atoi(e);
    // the selected product's form: scalar in place (phase_sel) or packed
    // (phase_sel_ct); QSB_JIT_SEL_FORM=ct / cs
    const char *sel_form = "phase_sel";
    if (const char *e = std::getenv("QSB_JIT_SEL_FORM"))
        if (!std::strcmp(e, "ct")) sel_form = "phase_sel_ct";
    // planar register layout (fused_dev.cuh: pphase / ppair): 0 (default:
    // measured slower on B200 — the packed results land in fresh register
    // pairs and ptxas copies them home around the uniform branches; QFT(30)
    // 34.0 -> 38.3 ms), 1 always, 2 for phase-dominated passes
    int planar_mode = 0;
    if (const char *e = std::getenv("QSB_JIT_PLANAR")) planar_mode = std::atoi(e);
    int nphase = 0;
    for (int o = 0; o < p.nops; ++o) nphase += p.ops[o].variant >= kPhaseVariant;
    const bool planar = planar_mode == 1 || (planar_mode == 2 && 2 * nphase > p.nops);
    if (planar) loop_run = 1 << 30;  // the op-table loops (run_phase / run_pair) are interleaved-layout code
    // Runs of >= tile_loop diagonal ops tested only on TILE bits (QFT rows:
    // the controls outside the tile) become one loop over the ops that
    // apply to this tile (a uniform bit mask), entries from a __constant__
    // table: no branch per op, skipped ops cost nothing, small code.  The
    // applicable ops run in circuit order, so the bits are unchanged.
    int tile_loop = 3;
    if (const char *e = std::getenv("QSB_JIT_TILE_LOOP")) tile_loop = std::atoi(e);
    // the loop body's complex product: packed (phase_ct: FMUL, FMUL, FFMA2
    // per amplitude; default) or scalar in place (QSB_JIT_LOOP_FORM=cs)
    const char *loop_form = "phase_ct";
    if (const char *e = std::getenv("QSB_JIT_LOOP_FORM"))
        if (!std::strcmp(e, "cs")) loop_form = "phase_cs";
    std::string consts;
    int nconst = 0;
    std::string src;
    src.reserve(8192 + (size_t)p.nops * 200);
    // QSB_JIT_TURNS=cs: combined runs multiply with the scalar in-place form
    if (const char *e = std::getenv("QSB_JIT_TURNS"))
        if (!std::strcmp(e, "cs")) src += "#define QSB_TURNS_SCALAR 1\n";
    src += "#include \"fused_dev.cuh\"\nusing namespace qsb;\nstruct GenProg {\n";
    src += planar ? "  static constexpr bool kPlanar = true;\n" : "  static constexpr bool kPlanar = false;\n";
    src += "  template <int RB>\n"
           "  static __device__ __forceinline__ void run(int s, const FStage &, const FOp *ops, uint32_t tid,\n"
           "      uint64_t base, float one, float4 (&v)[1 << RB]) {\n"
           // warp index and tile base through redux.sync: values ptxas knows
           // to be warp-uniform, so warp-bit and tile tests become uniform
           // branches (no BSSY / BSYNC reconvergence per op)
           "    const uint32_t wid = __reduce_or_sync(0xffffffffu, tid & ~31u);\n"
           "    const uint64_t ub = ((uint64_t)__reduce_or_sync(0xffffffffu, (unsigned)(base >> 32)) << 32) |\n"
           "                        __reduce_or_sync(0xffffffffu, (unsigned)base);\n"
           "    (void)wid;\n    (void)ub;\n    switch (s) {\n";
    char buf[256];
    int group_uniform = 1;  // QSB_JIT_GROUP=0: one branch per op
    if (const char *e = std::getenv("QSB_JIT_GROUP")) group_uniform = std::atoi(e);
    // One op as generated source.  grouped: the caller has already branched
    // on the op's warp-uniform test; only the lane part remains.
    // a gate entry: a literal of the generated source, or (parametric
    // programs) a load from the op table staged in shared memory, so a
    // circuit of the same structure with other angles reuses the program
    auto ent = [&](std::string &out, int oi, int i) {
        if (param) {
            out += "ops[" + std::to_string(oi) + "].m[" + std::to_string(i) + "]";
        } else {
            hexf(out, p.ops[oi].m[i]);
        }
    };
    auto emit_one = [&](int oi, bool grouped) -> std::string {
        const FOp &op = p.ops[oi];
        std::string out;
        char b[256];
        const std::string utest = grouped ? std::string() : uniform_test(op), ltest = lane_test(op);
        std::string test = utest;
        if (!ltest.empty()) test = test.empty() ? ltest : test + " && " + ltest;
        const bool in_branch = grouped || !utest.empty();
        const bool is_phase = op.variant >= kPhaseVariant;
        const int cls = is_phase ? -1 : (op.variant / 2) % 4;
        if (sel_mode && !ltest.empty() && (is_phase || cls == kSwap)) {
            // predicated selection under the lane test, branch only on the
            // (warp-uniform) rest
            out += utest.empty() ? "      {" : "      if (" + utest + ") {";
            if (is_phase) {
                const int R = (op.variant - kPhaseVariant) / 2, odd = (op.variant - kPhaseVariant) % 2;
                std::snprintf(b, sizeof b, " %s<%d, %s, RB>(%s, make_float2(",
                              planar ? (in_branch ? "pphase_sel_cs" : "pphase_sel") : sel_form, R,
                              odd ? "true" : "false", ltest.c_str());
                out += b;
                ent(out, oi, 6);
                out += ", ";
                ent(out, oi, 7);
                out += "), v); }\n";
            } else {
                const int slot = (op.variant / 2) / 4 - 1;
                std::snprintf(b, sizeof b, " %s<%d, %u, %s, RB>(%s, v); }\n", planar ? "pswap_sel" : "swap_sel", slot,
                              op.reg_need, op.half_need ? "true" : "false", ltest.c_str());
                out += b;
            }
            return out;
        }
        out += test.empty() ? "      {" : "      if (" + test + ") {";
        if (is_phase) {
            const int R = (op.variant - kPhaseVariant) / 2, odd = (op.variant - kPhaseVariant) % 2;
            const bool scalar = phase_mode == 2 || (phase_mode == 1 && (in_branch || !test.empty()));
            std::snprintf(b, sizeof b, " %s<%d, %s, RB>(make_float2(",
                          planar ? (in_branch || !test.empty() ? "pphase_cs" : "pphase")
                                 : (scalar ? "phase_cs" : "phase_ct"),
                          R, odd ? "true" : "false");
            out += b;
            ent(out, oi, 6);
            out += ", ";
            ent(out, oi, 7);
            out += "), v); }\n";
        } else {
            const int slot = (op.variant / 2) / 4 - 1;
            out += " const float m[8] = {";
            for (int i = 0; i < 8; ++i) {
                if (i) out += ", ";
                ent(out, oi, i);
            }
            std::snprintf(b, sizeof b, "}; %s<%d, %d, %u, %s, RB>(m, one, v); }\n", planar ? "ppair" : "pair_ct", slot,
                          cls, op.reg_need, op.half_need ? "true" : "false");
            out += b;
        }
        return out;
    };
    for (int k = 0; k < p.nstages; ++k) {
        const FStage &st = p.stages[k];
        std::snprintf(buf, sizeof buf, "    case %d: {\n", k);
        src += buf;
        for (int o = st.op_begin; o < st.op_end;) {
            const FOp &op = p.ops[o];
            // combined diagonal runs (QS_FUSED_COMBINE_PHASES, not bit-exact):
            // accumulate each op's angle (fixed-point turns, exact modular
            // sums) into one accumulator per register pattern under its
            // thread / tile predicate, then one complex product per amplitude
            uint32_t t0;
            if (p.combine && op.variant >= kPhaseVariant && unit_turns(op, &t0)) {
                int e2 = o;
                uint32_t tt;
                while (e2 < st.op_end && p.ops[e2].variant >= kPhaseVariant && unit_turns(p.ops[e2], &tt)) ++e2;
                if (e2 - o >= 2) {
                    std::vector<std::pair<uint32_t, uint32_t>> pats;  // (reg_need, half_need)
                    std::vector<uint32_t> cst;                      // folded unconditional turns
                    std::string adds;
                    for (int i = o; i < e2; ++i) {
                        const FOp &x = p.ops[i];
                        const std::pair<uint32_t, uint32_t> key(x.reg_need, x.half_need ? 1u : 0u);
                        size_t a = std::find(pats.begin(), pats.end(), key) - pats.begin();
                        if (a == pats.size()) {
                            pats.push_back(key);
                            cst.push_back(0);
                        }
                        unit_turns(x, &tt);
                        const std::string cond = op_test(x);
                        if (cond.empty()) {
                            cst[a] += tt;
                        } else {
                            std::snprintf(buf, sizeof buf, "        a%zu += (%s) ? 0x%08xu : 0u;\n", a, cond.c_str(), tt);
                            adds += buf;
                        }
                    }
                    std::snprintf(buf, sizeof buf, "      { // %d diagonal ops combined\n", e2 - o);
                    src += buf;
                    for (size_t a = 0; a < pats.size(); ++a) {
                        std::snprintf(buf, sizeof buf, "        uint32_t a%zu = 0x%08xu;\n", a, cst[a]);
                        src += buf;
                    }
                    src += adds;
                    const char *re[2] = {planar ? "x" : "x", planar ? "y" : "z"};
                    const char *im[2] = {planar ? "z" : "y", planar ? "w" : "w"};
                    // e^{i a} for each accumulator once per thread (one
                    // __sincosf each), and per distinct set of matching
                    // patterns the product of those factors (built from the
                    // set minus its last member, memoised): the SFU pipe
                    // (16 lanes / clk / SM) bounded QFT pass 0 when every
                    // amplitude took its own __sincosf.  Each factor is
                    // within ~4e-7 of e^{i a}; a product of m factors within
                    // ~m times that (the mode's bar is rtol 1e-5).
                    std::vector<std::vector<int>> sets;  // index = factor f<k>
                    std::string facs, muls;
                    auto factor = [&](auto &&self, const std::vector<int> &set) -> size_t {
                        size_t k = std::find(sets.begin(), sets.end(), set) - sets.begin();
                        if (k < sets.size()) return k;
                        if (set.size() == 1) {
                            std::snprintf(buf, sizeof buf, "        const float2 f%zu = turns_sincos(a%d);\n", sets.size(),
                                          set[0]);
                        } else {
                            const std::vector<int> head(set.begin(), set.end() - 1);
                            const size_t h = self(self, head), t = self(self, std::vector<int>{set.back()});
                            std::snprintf(buf, sizeof buf, "        const float2 f%zu = cmul_any(f%zu, f%zu);\n",
                                          sets.size(), h, t);
                        }
                        facs += buf;
                        sets.push_back(set);
                        return sets.size() - 1;
                    };
                    for (int j = 0; j < (1 << RB); ++j)
                        for (int h = 0; h < 2; ++h) {
                            std::vector<int> set;
                            for (size_t a = 0; a < pats.size(); ++a)
                                if (((uint32_t)j & pats[a].first) == pats[a].first && (!pats[a].second || h == 1))
                                    set.push_back((int)a);
                            if (set.empty()) continue;
                            const size_t e = factor(factor, set);
                            std::snprintf(buf, sizeof buf,
                                          "        if constexpr (%d < (1 << RB)) turns_apply(f%zu, v[%d].%s, v[%d].%s);\n",
                                          j, e, j, re[h], j, im[h]);
                            muls += buf;
                        }
                    src += facs;
                    src += muls;
                    src += "      }\n";
                    o = e2;
                    continue;
                }
            }
            auto tile_only = [&](const FOp &x) {
                return x.variant >= kPhaseVariant && x.ext_need != 0 && x.tid_need == 0 &&
                       x.reg_need == op.reg_need && x.half_need == op.half_need;
            };
            if (tile_loop > 0 && tile_only(op)) {
                int e2 = o;
                while (e2 < st.op_end && e2 - o < 32 && tile_only(p.ops[e2])) ++e2;
                const int len = e2 - o;
                if (len >= tile_loop && param) {  // entries from the op table
                    src += "      { uint32_t m = 0u;";
                    for (int i = 0; i < len; ++i) {
                        const unsigned long long E = p.ops[o + i].ext_need;
                        std::snprintf(buf, sizeof buf, " m |= (uint32_t)((ub & 0x%llxull) == 0x%llxull) << %d;", E, E, i);
                        src += buf;
                    }
                    std::snprintf(buf, sizeof buf,
                                  "\n        while (m) { const int i = __ffs(m) - 1; m &= m - 1u;"
                                  " %s<%d, %s, RB>(make_float2(ops[%d + i].m[6], ops[%d + i].m[7]), v); } }\n",
                                  planar ? "pphase" : loop_form, (int)op.reg_need, op.half_need ? "true" : "false", o, o);
                    src += buf;
                    o = e2;
                    continue;
                }
                if (len >= tile_loop) {
                    const int id = nconst++;
                    std::snprintf(buf, sizeof buf, "__constant__ unsigned kT%d[%d] = {", id, 2 * len);
                    consts += buf;
                    for (int i = 0; i < len; ++i) {
                        uint32_t bx, by;
                        std::memcpy(&bx, &p.ops[o + i].m[6], 4);
                        std::memcpy(&by, &p.ops[o + i].m[7], 4);
                        std::snprintf(buf, sizeof buf, "%s0x%08xu, 0x%08xu", i ? ", " : "", bx, by);
                        consts += buf;
                    }
                    consts += "};\n";
                    // applicable-op mask of this tile: consecutive single
                    // tile bits in ascending order are one shift
                    bool consecutive = true;
                    const int b0 = __builtin_ctzll(p.ops[o].ext_need);
                    for (int i = 0; i < len; ++i)
                        if (p.ops[o + i].ext_need != (1ull << (b0 + i))) consecutive = false;
                    src += "      { uint32_t m = ";
                    if (consecutive) {
                        std::snprintf(buf, sizeof buf, "(uint32_t)(ub >> %d) & 0x%xu;", b0,
                                      len == 32 ? 0xffffffffu : ((1u << len) - 1u));
                        src += buf;
                    } else {
                        src += "0u;";
                        for (int i = 0; i < len; ++i) {
                            const unsigned long long E = p.ops[o + i].ext_need;
                            std::snprintf(buf, sizeof buf, " m |= (uint32_t)((ub & 0x%llxull) == 0x%llxull) << %d;", E, E, i);
                            src += buf;
                        }
                    }
                    const int R = (int)op.reg_need;
                    std::snprintf(buf, sizeof buf,
                                  "\n        while (m) { const int i = __ffs(m) - 1; m &= m - 1u;"
                                  " %s<%d, %s, RB>(make_float2(__uint_as_float(kT%d[2 * i]), __uint_as_float(kT%d[2 * i + 1])), v); } }\n",
                                  planar ? "pphase" : loop_form, R, op.half_need ? "true" : "false", id, id);
                    src += buf;
                    o = e2;
                    continue;
                }
            }
            // optionally (QSB_JIT_LOOP_RUN, see kJitLoopRun) a long run of
            // one variant stays a loop over the shared-memory op table
            int e = o + 1;
            while (e < st.op_end && p.ops[e].variant == op.variant && p.ops[e].reg_need == op.reg_need &&
                   p.ops[e].half_need == op.half_need)
                ++e;
            // registers an op of this run touches (of 2^RB float4 per thread)
            const int touched = (1 << RB) >> __builtin_popcount(op.reg_need);
            if (e - o >= loop_run && touched >= kJitLoopMinRegs) {
                if (op.variant >= kPhaseVariant) {
                    const int R = (op.variant - kPhaseVariant) / 2, odd = (op.variant - kPhaseVariant) % 2;
                    std::snprintf(buf, sizeof buf, "      run_phase<%d, %s, RB>(ops + %d, %d, tid, base, v);\n", R,
                                  odd ? "true" : "false", o, e - o);
                } else {
                    const int cls = (op.variant / 2) % 4, slot = (op.variant / 2) / 4 - 1;
                    const bool need = (op.variant % 2) || cls == kCplx || cls == kSwap;
                    std::snprintf(buf, sizeof buf, "      run_pair<%d, %d, %s, RB>(ops + %d, %d, tid, base, v);\n",
                                  slot, cls, need ? "true" : "false", o, e - o);
                }
                src += buf;
                o = e;
                continue;
            }
            // one op per iteration (the next op may start a combined run or a
            // tile loop); consecutive ops under the SAME warp-uniform test
            // (a tile bit or warp bit) share one branch
            const std::string ut0 = uniform_test(op);
            int e3 = o + 1;
            if (group_uniform && !p.combine && !ut0.empty()) {
                auto loop_start = [&](int i) {
                    const FOp &x = p.ops[i];
                    if (!(tile_loop > 0 && x.variant >= kPhaseVariant && x.ext_need && !x.tid_need)) return false;
                    int k = i;
                    while (k < st.op_end && k - i < tile_loop && p.ops[k].variant >= kPhaseVariant &&
                           p.ops[k].ext_need && !p.ops[k].tid_need && p.ops[k].reg_need == x.reg_need &&
                           p.ops[k].half_need == x.half_need)
                        ++k;
                    return k - i >= tile_loop;
                };
                while (e3 < st.op_end && uniform_test(p.ops[e3]) == ut0 && !loop_start(e3)) ++e3;
            }
            if (e3 - o >= 2) {
                src += "      if (" + ut0 + ") {\n";
                for (; o < e3; ++o) src += emit_one(o, true);
                src += "      }\n";
            } else {
                src += emit_one(o, false);
                ++o;
            }
        }
        src += "    } break;\n";
    }
    src += "    default: break;\n    }\n  }\n";
    // The whole stage sequence with the stage layouts as literals (see
    // emit_run_stages).
    if (!planar && static_stages_enabled())
        emit_run_stages(src, p, RB, false);
    else
        src += "  static constexpr bool kOwnsStages = false;\n";
    std::snprintf(buf, sizeof buf,
                  "};\n"
                  "extern \"C\" __global__ void __maxnreg__(%d) qsb_pass(float4 *__restrict__ amps,\n"
                  "    const __grid_constant__ FParams p) {\n  fused_body<%d, %d, GenProg>(amps, p);\n}\n",
                  RB == 4 ? 168 : 96, K, RB);
    src += buf;
    if (!consts.empty()) {  // the constant tables go before the program that reads them
        const std::string head = "using namespace qsb;\n";
        const size_t at = src.find(head) + head.size();
        src.insert(at, consts);
    }
    return src;
}

// complex128 registers: every op straight-line (pair_ct_d / phase_ct_d) with
// its fp64 entries as literals from the caller's qs_op64 list (FOp k of the
// group is op `first + k`).
void hexd(std::string &out, double x) {
    uint64_t b;
    std::memcpy(&b, &x, 8);
    char buf[48];
    std::snprintf(buf, sizeof buf, "__longlong_as_double(0x%016llxll)", (unsigned long long)b);
    out += buf;
}

std::string generate_d(const FParams &p, int K, int RB, const qs_op64 *ops64) {
    std::string src;
    src.reserve(8192 + (size_t)p.nops * 400);
    src += "#include \"fused_dev.cuh\"\nusing namespace qsb;\nstruct GenProg {\n"
           "  static constexpr bool kPlanar = false;\n  template <int RB>\n"
           "  static __device__ __forceinline__ void run(int s, const FStage &, const FOp *, uint32_t tid,\n"
           "      uint64_t base, float, double2 (&v)[1 << RB]) {\n"
           "    const uint32_t wid = __reduce_or_sync(0xffffffffu, tid & ~31u);\n"
           "    const uint64_t ub = ((uint64_t)__reduce_or_sync(0xffffffffu, (unsigned)(base >> 32)) << 32) |\n"
           "                        __reduce_or_sync(0xffffffffu, (unsigned)base);\n"
           "    (void)wid;\n    (void)ub;\n    switch (s) {\n";
    char buf[256];
    for (int k = 0; k < p.nstages; ++k) {
        const FStage &st = p.stages[k];
        std::snprintf(buf, sizeof buf, "    case %d: {\n", k);
        src += buf;
        for (int o = st.op_begin; o < st.op_end; ++o) {
            const FOp &op = p.ops[o];
            const qs_op64 &g = ops64[o];
            std::string test = op_test(op);
            src += test.empty() ? "      {" : "      if (" + test + ") {";
            if (op.variant >= kPhaseVariant) {
                std::snprintf(buf, sizeof buf, " phase_ct_d<%u, RB>(make_double2(", op.reg_need);
                src += buf;
                hexd(src, g.m[6]);
                src += ", ";
                hexd(src, g.m[7]);
                src += "), v); }\n";
            } else {
                const int slot = (op.variant / 2) / 4 - 1;
                src += " const double m[8] = {";
                for (int i = 0; i < 8; ++i) {
                    if (i) src += ", ";
                    hexd(src, g.m[i]);
                }
                std::snprintf(buf, sizeof buf, "}; pair_ct_d<%d, %u, RB>(m, v); }\n", slot, op.reg_need);
                src += buf;
            }
        }
        src += "    } break;\n";
    }
    src += "    default: break;\n    }\n  }\n";
    if (static_stages_enabled())
        emit_run_stages(src, p, RB, true);
    else
        src += "  static constexpr bool kOwnsStages = false;\n";
    std::snprintf(buf, sizeof buf,
                  "};\n"
                  "extern \"C\" __global__ void __maxnreg__(%d) qsb_pass(float4 *__restrict__ amps,\n"
                  "    const __grid_constant__ FParams p) {\n  fused_body<%d, %d, GenProg, double2>(amps, p);\n}\n",
                  RB == 4 ? 168 : 96, K, RB);
    src += buf;
    return src;
}

// ---- compile service ------------------------------------------------------------
// NVRTC runs on a small pool of host worker threads; a finished cubin is
// loaded into the device context by the next launching thread that asks for
// it (or by qs_jit_sync), so no host thread blocks on a compile unless the
// caller asks for it (QSB_FUSED_JIT=2, qs_jit_sync).
struct Job;
bool compile_nvrtc(Job &job);
const char *const kNvrtcOpts[4] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "-DQSB_JIT=1"};

struct Job {
    int device = 0;
    std::string src;
    size_t smem_max = 0;
    int state = 0;  // 0 queued / compiling, 1 cubin ready, 2 failed
    std::vector<char> cubin;
    std::string err;
};
using Key = std::pair<int, std::string>;

std::mutex g_mu;
std::condition_variable g_cv;       // job state changes and new work
std::map<Key, CUfunction> g_fns;   // loaded programs
std::map<Key, bool> g_failed;
std::map<Key, std::shared_ptr<Job>> g_jobs;  // queued, compiling or awaiting load
std::deque<std::shared_ptr<Job>> g_queue;
std::vector<pthread_t> g_workers;
bool g_stop = false;

int jit_mode() {
    const char *e = std::getenv("QSB_FUSED_JIT");
    if (!e || !*e) return 1;
    return std::atoi(e);
}

// On-disk cache of compiled pass programs: a process that runs a circuit
// compiled before (same generated source, same options) loads the cubin
// instead of recompiling.  File = [u64 source length][source][cubin], so a
// hash collision is detected by comparing the source.  Directory:
// QSB_JIT_CACHE_DIR, else $XDG_CACHE_HOME/qsb200-jit or ~/.cache/qsb200-jit;
// QSB_JIT_CACHE=0 disables it.
std::string cache_path(const std::string &src) {
    const char *off = std::getenv("QSB_JIT_CACHE");
    if (off && *off == '0') return "";
    std::string dir;
    if (const char *d = std::getenv("QSB_JIT_CACHE_DIR")) {
        dir = d;
    } else if (const char *x = std::getenv("XDG_CACHE_HOME")) {
        dir = std::string(x) + "/qsb200-jit";
    } else if (const char *h = std::getenv("HOME")) {
        dir = std::string(h) + "/.cache/qsb200-jit";
    } else {
        return "";
    }
    uint64_t hsh = 1469598103934665603ull;  // FNV-1a over the source + the target
    for (unsigned char c : src) hsh = (hsh ^ c) * 1099511628211ull;
    char name[40];
    std::snprintf(name, sizeof name, "/%016llx.bin", (unsigned long long)hsh);
    return dir + name;
}

bool cache_load(const std::string &path, const std::string &src, std::vector<char> &cubin) {
    if (path.empty()) return false;
    FILE *f = std::fopen(path.c_str(), "rb");
    if (!f) return false;
    bool ok = false;
    uint64_t len = 0;
    if (std::fread(&len, 8, 1, f) == 1 && len == src.size()) {
        std::string got(len, '\0');
        if (std::fread(&got[0], 1, len, f) == len && got == src) {
            std::vector<char> rest;
            char buf[65536];
            size_t k;
            while ((k = std::fread(buf, 1, sizeof buf, f)) > 0) rest.insert(rest.end(), buf, buf + k);
            if (!rest.empty()) {
                cubin.swap(rest);
                ok = true;
            }
        }
    }
    std::fclose(f);
    return ok;
}

void cache_store(const std::string &path, const std::string &src, const std::vector<char> &cubin) {
    if (path.empty()) return;
    const size_t slash = path.rfind('/');
    const std::string dir = path.substr(0, slash);
    for (size_t i = 1; i <= dir.size(); ++i)  // mkdir -p
        if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
    const std::string tmp = path + ".tmp" + std::to_string((unsigned long long)pthread_self());
    FILE *f = std::fopen(tmp.c_str(), "wb");
    if (!f) return;
    const uint64_t len = src.size();
    bool ok = std::fwrite(&len, 8, 1, f) == 1 && std::fwrite(src.data(), 1, len, f) == len &&
              std::fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
    ok = std::fclose(f) == 0 && ok;
    if (ok)
        std::rename(tmp.c_str(), path.c_str());
    else
        std::remove(tmp.c_str());
}

// the cache key: the generated source plus the device headers it includes
// and the NVRTC options (a rebuilt library with changed headers or options
// must not load stale programs)
std::string cache_key(const std::string &src) {
    static const std::string tag = [] {
        uint64_t h = 1469598103934665603ull;
        for (const char *t : {kJitCommon, kJitFusedDev, kNvrtcOpts[0], kNvrtcOpts[1], kNvrtcOpts[2], kNvrtcOpts[3]})
            for (const char *c = t; *c; ++c) h = (h ^ (unsigned char)*c) * 1099511628211ull;
        char b[80];  // the compiler version too: programs differ between NVRTC releases
        std::snprintf(b, sizeof b, "\n// headers+options %016llx nvrtc %d.%d\n", (unsigned long long)h,
                      nvrtc().major, nvrtc().minor);
        return std::string(b);
    }();
    return src + tag;
}

std::atomic<unsigned long long> g_compiled{0}, g_cache_hits{0}, g_compile_failed{0};

bool compile_cubin(Job &job) {
    const std::string key = cache_key(job.src);
    const std::string cpath = cache_path(key);
    if (cache_load(cpath, key, job.cubin)) {
        ++g_cache_hits;
        return true;
    }
    const bool ok = compile_nvrtc(job);
    if (ok) {
        ++g_compiled;
        cache_store(cpath, key, job.cubin);
    } else {
        ++g_compile_failed;
    }
    return ok;
}

bool compile_nvrtc(Job &job) {
    const Nvrtc &nv = nvrtc();
    if (const char *dir = std::getenv("QSB_JIT_DUMP")) {  // generated sources, for offline SASS study
        uint64_t h = 1469598103934665603ull;
        for (char c : job.src) h = (h ^ (unsigned char)c) * 1099511628211ull;
        char name[48];
        std::snprintf(name, sizeof name, "/qsb_pass_%016llx.cu", (unsigned long long)h);
        const std::string path = std::string(dir) + name;
        if (FILE *f = std::fopen(path.c_str(), "w")) {
            std::fwrite(job.src.data(), 1, job.src.size(), f);
            std::fclose(f);
        }
    }
    const char *hdrs[2] = {kJitCommon, kJitFusedDev};
    const char *names[2] = {"common.cuh", "fused_dev.cuh"};
    nvrtcProgram_t prog = nullptr;
    if (nv.create(&prog, job.src.c_str(), "qsb_pass.cu", 2, hdrs, names) != 0) {
        job.err = "nvrtcCreateProgram failed";
        return false;
    }
    const char *opts[] = {kNvrtcOpts[0], kNvrtcOpts[1], kNvrtcOpts[2], kNvrtcOpts[3]};
    if (nv.compile(prog, 4, opts) != 0) {
        size_t n = 0;
        nv.log_size(prog, &n);
        std::string log(n, '\0');
        nv.log(prog, &log[0]);
        job.err = "NVRTC compile failed: " + log.substr(0, 2000);
        nv.destroy(&prog);
        return false;
    }
    size_t n = 0;
    nv.cubin_size(prog, &n);
    job.cubin.resize(n);
    nv.cubin(prog, job.cubin.data());
    nv.destroy(&prog);
    return true;
}

void *worker(void *) {
    std::unique_lock<std::mutex> lock(g_mu);
    for (;;) {
        g_cv.wait(lock, [] { return g_stop || !g_queue.empty(); });
        if (g_stop) return nullptr;
        std::shared_ptr<Job> job = g_queue.front();
        g_queue.pop_front();
        lock.unlock();
        const bool ok = compile_cubin(*job);
        lock.lock();
        job->state = ok ? 1 : 2;
        g_cv.notify_all();
    }
}

// Stop the workers: queued compiles are dropped, an in-flight one finishes,
// then the threads are joined.  Called by the Python layer's atexit hook
// (qs_jit_shutdown) before interpreter and library teardown: a compile
// running while libraries are torn down crashes, and joining from inside the
// dynamic loader's exit processing can deadlock with NVRTC's own dlopen.
void shutdown_workers() {
    std::vector<pthread_t> ws;
    {
        std::lock_guard<std::mutex> lock(g_mu);
        g_stop = true;
        for (auto &j : g_queue) j->state = 2;  // dropped
        g_queue.clear();
        ws.swap(g_workers);
    }
    g_cv.notify_all();
    for (pthread_t t : ws) pthread_join(t, nullptr);
}

void ensure_workers() {  // g_mu held; libnvrtc is loaded (jit_enabled)
    if (!g_workers.empty() || g_stop) return;
    unsigned n = std::thread::hardware_concurrency();
    n = n < 2 ? 1 : (n > 16 ? 8 : n / 2);
    if (const char *w = std::getenv("QSB_JIT_WORKERS")) n = (unsigned)std::max(1, std::atoi(w));
    // NVRTC recurses deeply on long straight-line programs: give the workers
    // the stack a main thread would have and then some (virtual reservation)
    pthread_attr_t attr;
    pthread_attr_init(&attr);
    pthread_attr_setstacksize(&attr, (size_t)512 << 20);
    for (unsigned i = 0; i < n; ++i) {
        pthread_t t;
        if (pthread_create(&t, &attr, worker, nullptr) == 0) g_workers.push_back(t);
    }
    pthread_attr_destroy(&attr);
}

// Load a compiled job into the current device context (g_mu held).
CUfunction load(const Key &key, Job &job) {
    const Driver &dr = driver();
    CUmodule mod = nullptr;
    CUfunction fn = nullptr;
    if (dr.load(&mod, job.cubin.data()) != CUDA_SUCCESS || dr.get(&fn, mod, "qsb_pass") != CUDA_SUCCESS) {
        job.err = "cuModuleLoadData / cuModuleGetFunction failed";
        fn = nullptr;
    } else if (dr.set_attr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)job.smem_max) !=
               CUDA_SUCCESS) {
        job.err = "cuFuncSetAttribute(max dynamic smem) failed";
        fn = nullptr;
    }
    if (fn) {
        g_fns[key] = fn;
    } else {
        g_failed[key] = true;
        if (std::getenv("QSB_FUSED_JIT_VERBOSE")) std::fprintf(stderr, "qsb jit: %s\n", job.err.c_str());
    }
    return fn;
}

}  // namespace

// Should fused passes use compiled programs at all (policy, NVRTC present)?
bool jit_enabled() { return jit_mode() > 0 && nvrtc().ok && driver().ok; }

// Register bits per thread of compiled programs: QSB_FUSED_JIT_RB (3 or 4)
// or the caller's choice (5 bits = 4 compute warps per SM measured slower).
int jit_rb(int dflt) {
    const char *e = std::getenv("QSB_FUSED_JIT_RB");
    if (e && *e == '3') return 3;
    if (e && *e == '4') return 4;
    return dflt == 3 ? 3 : 4;
}

// The compiled program for one planned launch group, or nullptr while it is
// still compiling (the compile is queued on first request) or if it cannot be
// built.  wait = true blocks until the compile has finished (policy 2).
// Parametric programs (QSB_JIT_PARAMETRIC: 1 = auto, the default; 2 =
// always; 0 = never).  A literal program bakes the gate entries in (fastest:
// immediate operands); a parametric one reads them from the op table, so
// every circuit of the same STRUCTURE (op kinds, slots, classes, masks) runs
// it — a variational loop changing only angles compiles nothing new.  Auto:
// once a second distinct literal program of one structure is requested, that
// structure switches to its parametric program.
std::map<Key, std::set<size_t>> g_struct_lits;  // parametric key -> hashes of the literal sources seen (g_mu)

int param_policy() {
    const char *e = std::getenv("QSB_JIT_PARAMETRIC");
    return e && *e ? std::atoi(e) : 1;
}

// The key to run for this launch group: the literal program, or the
// parametric one of its structure (g_mu held).
Key choose_key(int device, const FParams &p, int K, int RB, bool *is_param) {
    *is_param = false;
    Key lit(device, generate(p, K, RB, false));
    const int pol = param_policy();
    if (pol == 0 || p.combine) return lit;
    if (g_fns.count(lit) && pol == 1) return lit;
    Key par(device, generate(p, K, RB, true));
    if (pol == 2 || g_fns.count(par)) {
        *is_param = true;
        return par;
    }
    std::set<size_t> &seen = g_struct_lits[par];
    seen.insert(std::hash<std::string>()(lit.second));
    if (seen.size() >= 2) {
        *is_param = true;
        return par;
    }
    return lit;
}

void *jit_get(int device, const FParams &p, int K, int RB, size_t smem_max, bool wait,
              const qs_op64 *ops64) {
    Key key;
    if (ops64) {
        key = Key(device, generate_d(p, K, RB, ops64));
    } else {
        std::lock_guard<std::mutex> lock(g_mu);
        bool is_param = false;
        key = choose_key(device, p, K, RB, &is_param);
    }
    if (const char *dir = std::getenv("QSB_FUSED_JIT_DUMP")) {  // tooling: keep the generated sources
        static int count = 0;
        const std::string path = std::string(dir) + "/qsb_pass_" + std::to_string(count++) + ".cu";
        if (FILE *f = std::fopen(path.c_str(), "w")) {
            std::fputs(key.second.c_str(), f);
            std::fclose(f);
        }
    }
    std::unique_lock<std::mutex> lock(g_mu);
    auto it = g_fns.find(key);
    if (it != g_fns.end()) return (void *)it->second;
    if (g_failed.count(key)) return nullptr;
    if (g_stop) return nullptr;  // shutting down: interpreter only
    std::shared_ptr<Job> &job = g_jobs[key];
    if (!job) {
        job = std::make_shared<Job>();
        job->device = device;
        job->src = key.second;
        job->smem_max = smem_max;
        // a program in the on-disk cache is loaded right away (a file read),
        // so even the first launch of a known pass runs compiled
        const std::string ck = cache_key(job->src);
        if (cache_load(cache_path(ck), ck, job->cubin)) {
            ++g_cache_hits;
            job->state = 1;
        } else {
            ensure_workers();
            g_queue.push_back(job);
            g_cv.notify_all();
        }
    }
    std::shared_ptr<Job> j = job;
    if (wait) g_cv.wait(lock, [&] { return j->state != 0; });
    if (j->state == 0) return nullptr;
    g_jobs.erase(key);
    if (j->state == 2) {
        g_failed[key] = true;
        if (std::getenv("QSB_FUSED_JIT_VERBOSE")) std::fprintf(stderr, "qsb jit: %s\n", j->err.c_str());
        return nullptr;
    }
    return (void *)load(key, *j);
}

// An already loaded program, without queueing or loading anything (used while
// the stream is being recorded into a CUDA graph).
void *jit_lookup(int device, const FParams &p, int K, int RB, const qs_op64 *ops64) {
    std::lock_guard<std::mutex> lock(g_mu);
    if (ops64) {
        auto it = g_fns.find(Key(device, generate_d(p, K, RB, ops64)));
        return it == g_fns.end() ? nullptr : (void *)it->second;
    }
    auto it = g_fns.find(Key(device, generate(p, K, RB, false)));
    if (it != g_fns.end()) return (void *)it->second;
    if (param_policy() != 0 && !p.combine) {
        it = g_fns.find(Key(device, generate(p, K, RB, true)));
        if (it != g_fns.end()) return (void *)it->second;
    }
    return nullptr;
}

// Wait for every queued compile and load the programs of `device` (< 0: the
// current device's).  Returns the number of programs that failed.
int jit_sync(int device) {
    std::unique_lock<std::mutex> lock(g_mu);
    g_cv.wait(lock, [] {
        for (auto &kv : g_jobs)
            if (kv.second->state == 0) return false;
        return true;
    });
    int failed = 0;
    for (auto it = g_jobs.begin(); it != g_jobs.end();) {
        if (device >= 0 && it->first.first != device) {
            ++it;
            continue;
        }
        if (it->second->state == 1) {
            DeviceGuard guard(it->first.first);
            if (!load(it->first, *it->second)) ++failed;
        } else {
            g_failed[it->first] = true;
            ++failed;
        }
        it = g_jobs.erase(it);
    }
    return failed;
}

int jit_launch(qs_state *s, void *fn, const FParams &p, size_t smem, unsigned grid, unsigned block) {
    float4 *amps = (float4 *)s->amps;
    void *args[2] = {(void *)&amps, (void *)&p};
    if (driver().launch((CUfunction)fn, grid, 1, 1, block, 1, 1, (unsigned)smem, (CUstream)s->stream, args,
                        nullptr) != CUDA_SUCCESS)
        return set_error(QS_ERR_CUDA, "cuLaunchKernel of a compiled pass failed");
    return QS_OK;
}


}  // namespace qsb

extern "C" int qs_jit_sync(int device) {
    const int failed = qsb::jit_sync(device);
    return failed ? qsb::set_error(QS_ERR_CUDA, std::to_string(failed) + " pass program(s) failed to compile")
                  : QS_OK;
}

extern "C" int qs_jit_stats(uint64_t *compiled, uint64_t *cache_hits, uint64_t *failed) {
    if (compiled) *compiled = qsb::g_compiled.load();
    if (cache_hits) *cache_hits = qsb::g_cache_hits.load();
    if (failed) *failed = qsb::g_compile_failed.load();
    return QS_OK;
}

extern "C" int qs_jit_shutdown(void) {
    qsb::shutdown_workers();
    return QS_OK;
}
