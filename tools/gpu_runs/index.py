#!/usr/bin/env python3
"""Regenerate the index in tools/gpu_runs/README.md from each command file's
first comment line."""
import glob
import os

HERE = os.path.dirname(os.path.abspath(__file__))
HEAD = """# tools/gpu_runs/

Command files of individual `gpurun` calls, kept so every number quoted in
DESIGN.md and profiles/ can be re-run:
`/usr/local/graft/bin/gpurun -- 'bash tools/gpu_runs/<round>/<file>'`.
Each file's first comment line says what it measured; the index below is
generated from those lines (`python tools/gpu_runs/index.py`).
"""


def first_comment(path):
    """the first comment line, else the first command (uncommented files)"""
    cmd = ""
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line.startswith("#") and not line.startswith("#!"):
                return line.lstrip("# ").strip()
            if line and not line.startswith("#") and not line.startswith("set ") and not cmd:
                cmd = line
    return f"(no comment) `{cmd[:110]}`" if cmd else ""


def main():
    lines = [HEAD]
    for rnd in sorted(d for d in os.listdir(HERE) if os.path.isdir(os.path.join(HERE, d))):
        files = sorted(glob.glob(os.path.join(HERE, rnd, "*.sh")))
        lines.append(f"## {rnd} ({len(files)} files)\n")
        lines.append("| file | what it measured |")
        lines.append("|---|---|")
        for p in files:
            lines.append(f"| `{rnd}/{os.path.basename(p)}` | {first_comment(p).replace('|', '/')} |")
        lines.append("")
    with open(os.path.join(HERE, "README.md"), "w") as f:
        f.write("\n".join(lines))


if __name__ == "__main__":
    main()
