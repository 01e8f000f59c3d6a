"""Regenerate tests/golden/campaign/ref_trace.jsonl and ref_report.json: the
UNMODIFIED reference run_campaign (pipeline.cpp:357-590, through
oracle/_ref/libvsref.so) on campaign/campaign_100.json.

    python tests/golden/make_campaign_golden.py
"""
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref as R  # noqa: E402


def main():
    camp = os.path.join(HERE, "campaign")
    with tempfile.TemporaryDirectory() as tmp:
        R.run_campaign(os.path.join(camp, "campaign_100.json"), os.path.join(camp, "ref_trace.jsonl"),
                       os.path.join(camp, "ref_report.json"), os.path.join(tmp, "fep.tsv"))


if __name__ == "__main__":
    main()
