"""Merge tools/cpu_pin.py outputs into profiles/cpu_pin.json (bench.py's
`model_validation`): per workload the full reference run, the model, and the
model's error, with the conditions of each run.

    python tools/pin_summary.py out.json clean.jsonl[:note] [more.jsonl[:note] ...]
"""
import json
import sys


def main(out, inputs):
    runs = []
    seen = set()  # (workload, threads): the first input that has it wins
    for spec in inputs:
        path, _, note = spec.partition(":")
        for line in open(path):
            line = line.strip()
            if not line.startswith("{"):
                continue
            d = json.loads(line)
            key = (d["workload"], d.get("threads"))
            if key in seen:
                continue
            seen.add(key)
            runs.append({"workload": d["workload"], "threads": d.get("threads"),
                         "measured_ms": d["measured_ms"], "model_ms": d["model_ms"],
                         "model_error": d["model_error"], "source": path, "conditions": note})
    doc = {"what": "full reference UnitarySimulator::simulate_full_state ('unitary-parallel') on the GPU box's "
                   "host vs bench.py's component model (cpu_sample_circuit, allow_full=False), same threads",
           "runs": runs,
           "max_abs_error": max(abs(r["model_error"]) for r in runs) if runs else None}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
