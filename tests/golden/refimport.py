"""Import the read-only reference package (this container only).

The reference snapshot lacks ``samp/tokenization.py``.  We stage a copy of
``/root/reference/pkg/src/samp`` under a temp dir (never inside the repo),
drop in our restated tokenizer, and import it as ``samp``.  Used only by the
golden-vector generator; nothing on the GPU box imports this.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile

REF_SRC = "/root/reference/pkg/src/samp"
_HERE = os.path.dirname(os.path.abspath(__file__))
_TOKENIZER = os.path.join(_HERE, "..", "..", "paper_2209_09130_b200", "tokenization.py")


def load_reference():
    if not os.path.isdir(REF_SRC):
        raise RuntimeError("reference tree not present (golden generation runs in the build container)")
    stage = tempfile.mkdtemp(prefix="samp_ref_")
    dst = os.path.join(stage, "samp")
    shutil.copytree(REF_SRC, dst)
    with open(_TOKENIZER, encoding="utf-8") as fh:
        src = fh.read()
    # our tokenizer imports .errors, which the reference also provides
    with open(os.path.join(dst, "tokenization.py"), "w", encoding="utf-8") as fh:
        fh.write(src)
    sys.path.insert(0, stage)
    for name in list(sys.modules):
        if name == "samp" or name.startswith("samp."):
            del sys.modules[name]
    import samp  # noqa: F401

    return samp
