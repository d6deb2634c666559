"""SASS evidence for profiles/: instruction mix of the non-timed step kernel, its
TMA / mbarrier / cp.async instructions, and the fall-through path of one in-range
level pair of the 8-slot unrolled loop (mbarrier wait .. arrive).

usage: python tools/sass_summary.py [OUT] [grid|ws]   (reads paper_1310_4218_b200/libod_b200.so)
"""
import collections
import re
import subprocess
import sys

_ARGS = "EEEvPKNS_8ChunkDevEPKNS_7TileDevEiiPKdiiiiPyPKyiyS9_NS_8PackArgsENS_8StepDepsE"
KERNELS = {
    "grid": ("_ZN3odb16column_step_gridILi6ELb0ELi4ELi8" + _ARGS, "column_step_grid<6,false,4,8>"),
    "ws": ("_ZN3odb14column_step_wsILi6ELb0ELi3" + _ARGS, "column_step_ws<6,false,3>"),
}


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "profiles/r2_sass_column_step_grid.txt"
    kernel, label = KERNELS[sys.argv[2] if len(sys.argv) > 2 else "grid"]
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", kernel, "paper_1310_4218_b200/libod_b200.so"],
                          check=True, capture_output=True, text=True).stdout
    ins, pos = [], {}
    for line in sass.splitlines():
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            pos[int(m.group(1), 16)] = len(ins)
            ins.append((int(m.group(1), 16), m.group(2).strip()))

    def op(s):
        return (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0]

    mix = collections.Counter(op(s) for _, s in ins)
    out = ["# cuobjdump -sass paper_1310_4218_b200/libod_b200.so, kernel "
           f"{label} (sm_100a)", "# instruction mix:"]
    out += [f"{v:7d} {k}" for k, v in mix.most_common(32)]
    out.append("# TMA (UTMALDG), mbarrier (SYNCS), cp.async (LDGSTS) and proxy fences (first 80):")
    keep = ("UTMALDG", "SYNCS", "LDGSTS", "FENCE", "ARRIVES")
    out += [f" /*{a:04x}*/ {s} ;" for a, s in ins if op(s) in keep][:80]
    waits = [i for i, (_, s) in enumerate(ins) if "PHASECHK" in s and re.search(r"\[UR\d+\]\s*,", s)]
    def pair_path(w):
        i, path = w, []
        while "SYNCS.ARRIVE" not in ins[i][1]:
            a, s = ins[i]
            m = re.match(r"BRA (0x[0-9a-f]+)", s)
            if m and i != w + 1:  # (w + 1: the wait's retry branch)
                i = pos[int(m.group(1), 16)]
                continue
            path.append((a, s))
            i += 1
        path.append(ins[i])
        return path

    if len(waits) < 9:  # (a kernel without the interleaved tile's pair layout)
        open(out_path, "w").write("\n".join(out) + "\n")
        print(out[2])
        return
    # waits[3..8]: the six in-range pair bodies (P0 first / other, P1, P2, P3 last / other)
    bodies = [pair_path(w) for w in waits[3:9]]
    fps = [sum(op(s) in ("DADD", "DFMA", "DMUL") for _, s in b) for b in bodies]
    out.append("# in-range level pairs of the 8-slot unrolled loop (mbarrier wait .. arrive, "
               "fall-through path), instructions / of which not FP64: "
               + ", ".join(f"{len(b)}/{len(b) - f}" for b, f in zip(bodies, fps)))
    path = bodies[2]
    out.append(f"# the pair at slots 2,3 ({len(path)} instructions):")
    out += [f" /*{a:04x}*/ {s} ;" for a, s in path]
    open(out_path, "w").write("\n".join(out) + "\n")
    print(out[-len(path) - 2])


if __name__ == "__main__":
    main()
