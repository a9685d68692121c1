"""Shared fixtures: golden vectors (produced by running the reference, see
tests/golden/make_golden.py), markers, and GPU availability."""

import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if path.endswith(".gz"):
        with gzip.open(path, "rt") as fh:
            return json.load(fh)
    with open(path) as fh:
        return json.load(fh)


def golden_dict_bytes(name="default.zsd"):
    with open(os.path.join(GOLDEN, "dicts", name), "rb") as fh:
        return fh.read()


@pytest.fixture(scope="session")
def codec_cases():
    return load_golden("codec_cases.json.gz")


@pytest.fixture(scope="session")
def decode_cases():
    return load_golden("decode_cases.json.gz")


@pytest.fixture(scope="session")
def preprocess_cases():
    return load_golden("preprocess_cases.json.gz")


@pytest.fixture(scope="session")
def stream_cases():
    return load_golden("stream_cases.json.gz")


@pytest.fixture(scope="session")
def corpus_hashes():
    return load_golden("corpus_hashes.json")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def train_cases():
    return load_golden("train_cases.json.gz")
