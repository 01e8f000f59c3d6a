"""Regenerate the SMZC codec fixtures from the UNMODIFIED reference codec
(oracle/_ref/libvsref.so: codec::compress_stream / train_dictionary,
codec.cpp:82-130, 254-267):

    python tests/golden/make_codec_golden.py

Writes tests/golden/codec/:
  library_100.smzc     campaign/sample_library_100.smi compressed with
                       campaign/smiles.dict (the reference's proj/data/smiles.dict,
                       copied verbatim: campaign_100.json names it)
  trained.dict         train_dictionary(sample library lines, 64) as SMZ1
  library_trained.smzc the sample library compressed with trained.dict
"""
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref as R  # noqa: E402


def main():
    out = os.path.join(HERE, "codec")
    os.makedirs(out, exist_ok=True)
    d = os.path.join(HERE, "campaign", "smiles.dict")
    shutil.copyfile("/root/reference/proj/data/smiles.dict", d)
    text = open(os.path.join(HERE, "campaign", "sample_library_100.smi"), "rb").read()
    open(os.path.join(out, "library_100.smzc"), "wb").write(R.smzc_compress(text, d))
    trained = R.train_dictionary(text, 64)
    td = os.path.join(out, "trained.dict")
    open(td, "wb").write(trained)
    open(os.path.join(out, "library_trained.smzc"), "wb").write(R.smzc_compress(text, td))


if __name__ == "__main__":
    main()
