"""Build tuning variants of the library (-D defines) and time cfg builds with each.

    python tools/tune.py build            # here (CPU): compile variants into tune_variants/
    python tools/tune.py run 3 4          # on the GPU box: time configs with every variant
"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.environ.get("TUNE_DIR", os.path.join(ROOT, "tune_variants"))
VARIANTS = {
    "base": [],
    "stage8": ["WT_WG_STAGE8=1"],
    "e32_2": ["WT_WG_E32=2"],
}
if os.environ.get("TUNE_ONLY"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["TUNE_ONLY"].split(",")}
CPW = os.environ.get("TUNE_CPW", "16").split(",")
if sys.argv[1] == "build":
    from paper_1407_8142_b200 import _build
    os.makedirs(VDIR, exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor
    def one(item):
        name, defs = item
        _build.build(force=True, defines=defs, out=os.path.join(VDIR, f"lib_{name}.so"))
        return name
    with ThreadPoolExecutor(len(VARIANTS)) as ex:
        for name in ex.map(one, VARIANTS.items()):
            print("built", name)
else:
    cfgs = sys.argv[2:] or ["4"]
    for name in VARIANTS:
      for cpw in CPW:
        env = dict(os.environ, WT_LIB_PATH=os.path.join(VDIR, f"lib_{name}.so"), WT_CHAINS_PER_WARP=cpw)
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "kprof.py"), *cfgs],
                             capture_output=True, text=True, env=env, timeout=600)
        lines = [l for l in out.stdout.splitlines() if l.startswith("cfg") or "k_group" in l]
        print(f"== {name} cpw={cpw}")
        print("\n".join(lines) if lines else out.stderr[-800:])
