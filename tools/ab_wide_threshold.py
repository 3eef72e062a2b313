"""ab_variants.py with blocks.WIDE_CTA_MAX_MEAN_ROW overridden (first argument): A/B of the wide-CTA hint on blocks the default threshold does not flag."""
import sys, runpy
sys.path.insert(0, "/root/repo")
import paper_2601_07628_b200.blocks as b
b.WIDE_CTA_MAX_MEAN_ROW = float(sys.argv.pop(1))
sys.argv[0] = "tools/ab_variants.py"
runpy.run_path("tools/ab_variants.py", run_name="__main__")
