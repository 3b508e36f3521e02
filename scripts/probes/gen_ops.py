"""Experiment: turn a QSB_FUSED_DUMP plan into a compile-time op program
(gen_ops.inc) for k_fused built with -DQSB_GEN_OPS."""
import sys
lines = open(sys.argv[1]).read().split("\n")
stages = []
for ln in lines:
    w = ln.split()
    if not w:
        continue
    if w[0] == "pass":
        if stages:
            break  # first pass only
    elif w[0] == "stage":
        stages.append([])
    elif w[0] == "op":
        stages[-1].append((int(w[1]), int(w[2])))
out = ["template <int RB>", "__device__ __forceinline__ void gen_ops(int s, const FOp *ops, uint32_t tid, uint64_t base, float4 (&v)[1 << RB]) {", "    switch (s) {"]
for k, ops in enumerate(stages):
    out.append(f"    case {k}:")
    for o, var in ops:
        if var >= 40:
            R, odd = (var - 40) // 2, (var - 40) % 2
            call = f"apply_phase<{R}, {'true' if odd else 'false'}, RB>(ops[{o}], v)"
        else:
            need = var % 2
            cls = (var // 2) % 4
            slot = (var // 2) // 4 - 1
            need_b = "true" if (need or cls in (0, 3)) else "false"
            call = f"apply_pair<{slot}, {cls}, {need_b}, RB>(ops[{o}], v)"
        out.append(f"        if (op_ok(ops[{o}], tid, base)) {call};")
    out.append("        break;")
out += ["    default: break;", "    }", "}"]
open(sys.argv[2], "w").write("\n".join(out) + "\n")
print(len(stages), "stages", sum(len(s) for s in stages), "ops")
