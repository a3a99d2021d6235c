#!/usr/bin/env python
"""Static register-file read model of the force loop.

Hypothesis from scripts/ubench_operands.cu (profiles/r01_ubench_operands.txt): a packed
FP32x2 instruction occupies the FMA pipe for 2 cycles, but its source operands must be
read from the register file first, and a 64-bit register pair costs ~1 read-cycle, a
broadcast .F32 scalar ~0.6, the same pair read twice in one instruction ~2.8, an operand
served by the reuse cache (.reuse on the same register in the same slot of the previous
instruction) 0.  The loop body of the hottest backward branch is costed per
instruction; pred_frac_of_pipe = pipe cycles / max(pipe cycles, read cycles) is the FMA
pipe utilisation the loop could reach if register reads were the only other limit.

  cuobjdump -sass paper_2509_19294_b200/libnbody.so > /tmp/f.sass
  python scripts/rf_model.py /tmp/f.sass [kernel-name-substring] [--list]
"""
import os
import re
import sys

SAME = float(os.environ.get("SAME", "1.8"))   # extra cost of reading a pair already read by this instruction
SCAL = float(os.environ.get("SCAL", "0.6"))   # broadcast .F32 scalar operand
PACKED = re.compile(r"F(FMA|ADD|MUL)2")
OPND = re.compile(r"-?\|?(R\d+)(\.reuse)?(\.F32x2\.HI_LO|\.F32)?")


def instructions(func_text):
    out = []
    for ln in func_text.splitlines():
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            out.append((int(m.group(1), 16), m.group(2).strip()))
    return out


def loop_body(ins):
    """Instructions of the backward branch whose body holds the most packed FP32 ops."""
    best = None
    for a, t in ins:
        m = re.match(r"(@!?U?P\d+ )?BRA(\.U)?( !?UP\d+,)? (0x[0-9a-f]+)", t)
        if m and int(m.group(4), 16) < a:
            tgt = int(m.group(4), 16)
            body = [x for x in ins if tgt <= x[0] <= a]
            n = sum(1 for x in body if PACKED.match(x[1]))
            if best is None or n > best[0]:
                best = (n, body)
    return best[1] if best else []


def cost_of(body, listing=False):
    prev, rf, pipe, n2, mufu, other = {}, 0.0, 0, 0, 0, 0
    for _, t in body:
        op = t.split()[0]
        c_ins = 0.0
        if PACKED.match(op):
            n2 += 1
            pipe += 2
            ops = [o.strip() for o in t[len(op):].split(",")][1:]   # sources only
            now, seen = {}, set()
            for slot, o in enumerate(ops):
                m = OPND.match(o)
                if not m:
                    continue          # immediate
                reg, pair = m.group(1), (m.group(3) or "").startswith(".F32x2")
                c = 1.0 if pair else SCAL
                if prev.get(slot) == reg:
                    c = 0.0
                elif reg in seen:
                    c = SAME
                seen.add(reg)
                c_ins += c
                if m.group(2):
                    now[slot] = reg
            prev = now
            rf += c_ins
        else:
            prev = {}
            if op.startswith("MUFU"):
                mufu += 1
            else:
                other += 1
        if listing:
            print(f"{c_ins:4.1f}  {t}")
    return {"fp32x2": n2, "pipe_cycles": pipe, "rf_read_cycles": round(rf, 1), "mufu": mufu,
            "other": other, "pred_frac_of_pipe": round(pipe / max(pipe, rf, 1e-9), 4)}


def main():
    text = open(sys.argv[1]).read()
    want = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
    for f in re.split(r"\n\s+Function : ", text)[1:]:
        name = f.split("\n")[0]
        if want and want not in name:
            continue
        body = loop_body(instructions(f))
        print(name[-70:], cost_of(body, listing="--list" in sys.argv))


if __name__ == "__main__":
    main()
