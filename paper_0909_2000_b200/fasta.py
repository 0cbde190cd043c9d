"""FASTA input for the CLI — restates the reference reader (io.cpp:32-100).

Blank lines and trailing CR are skipped, '>' starts a record (header trimmed at
the right), sequence bytes are upper-cased, whitespace is ignored, and
non-printable bytes or '>' inside sequence data are errors, as are data before
the first header and records without sequence data.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

from .alignplot import Sequence


class ParseError(RuntimeError):
    """model.hpp:28-31."""


@dataclass
class FastaRecord:
    header: str
    sequence: bytearray


def read_fasta_bytes(data: bytes, source: str = "<memory>") -> List[FastaRecord]:
    records: List[FastaRecord] = []
    header_line = 0
    in_record = False
    for line_no, raw in enumerate(data.split(b"\n"), start=1):
        if raw.endswith(b"\r"):
            raw = raw[:-1]
        if not raw or raw.isspace():
            continue
        if raw[:1] == b">":
            if in_record and not records[-1].sequence:
                raise ParseError(f"{source}:{header_line}: record '{records[-1].header}' has no sequence data")
            records.append(FastaRecord(raw[1:].rstrip().decode("latin-1"), bytearray()))
            header_line = line_no
            in_record = True
            continue
        if not in_record:
            raise ParseError(f"{source}:{line_no}: sequence data before first header")
        for c in raw:
            if chr(c).isspace() and c < 128:
                continue
            if not (32 <= c < 127) or c == ord(">"):
                raise ParseError(f"{source}:{line_no}: unexpected byte in sequence data")
            records[-1].sequence.append(ord(chr(c).upper()) if 97 <= c <= 122 else c)
    if not records:
        raise ParseError(f"{source}: no FASTA records")
    if not records[-1].sequence:
        raise ParseError(f"{source}:{header_line}: record '{records[-1].header}' has no sequence data")
    return records


def read_fasta(path: str) -> List[FastaRecord]:
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise ParseError(f"{path}: cannot open file")
    return read_fasta_bytes(data, path)


def select_record(records: List[FastaRecord], name: str, source: str) -> FastaRecord:
    """io.cpp:78-95: exact header, or the header's first whitespace-delimited token."""
    if not name:
        return records[0]
    for rec in records:
        if rec.header == name:
            return rec
        cut = min([i for i in (rec.header.find(" "), rec.header.find("\t")) if i >= 0], default=-1)
        if cut >= 0 and rec.header[:cut] == name:
            return rec
    raise ParseError(f"{source}: no record named '{name}'")


def to_sequence(rec: FastaRecord) -> Sequence:
    return Sequence(rec.header, bytes(rec.sequence))
