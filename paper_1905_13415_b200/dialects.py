"""DFA tables handed to ``parpa_create_dfa`` (the parsing rules are the configuration).

Tables are row-per-group (tab:ttable): ``transition[g][s]`` is the state
entered from state ``s`` on a symbol of group ``g``; ``emit[g][s]`` is the emission
kind of that symbol (DATA / CTRL / FIELD / RECORD, by SOURCE state — reading R2);
``eoi[s]`` is the end-of-input action of final state ``s`` (reading R6).  Start state
is index 0 (reading R1).  The invalid state is absorbing.

This is product data, independent of ``oracle/`` (which hard-codes the same
languages as control flow); tests/test_dialect_tables.py proves the two agree.
"""
from __future__ import annotations

from dataclasses import dataclass, field

DATA, CTRL, FIELD, RECORD = 0, 1, 2, 3
EOI_NONE, EOI_RECORD, EOI_ERROR = 0, 1, 2
D, C, F, R = DATA, CTRL, FIELD, RECORD


@dataclass
class DfaTables:
    name: str
    states: list            # state names, index = state id
    groups: list            # list of bytes objects; the last group is the catch-all (empty)
    transition: list        # [G][S]
    emit: list              # [G][S]
    eoi: list               # [S]
    start: int = 0
    invalid: int = -1
    group_of_byte: list = field(default_factory=list)

    def __post_init__(self):
        if self.invalid < 0:
            self.invalid = len(self.states) - 1
        catch_all = len(self.groups) - 1
        gob = [catch_all] * 256
        for g, syms in enumerate(self.groups):
            for b in syms:
                gob[b] = g
        self.group_of_byte = gob

    @property
    def S(self):
        return len(self.states)

    @property
    def G(self):
        return len(self.groups)

    def as_dict(self):
        return {"group_of_byte": self.group_of_byte, "transition": self.transition, "emit": self.emit,
                "eoi": self.eoi, "start": self.start, "invalid": self.invalid}


def rfc4180() -> DfaTables:
    """RFC 4180 CSV with LF record delimiters: tab:ttable, six states incl. INV."""
    EOR, ENC, FLD, EOF, ESC, INV = range(6)
    return DfaTables(
        "csv", ["EOR", "ENC", "FLD", "EOF", "ESC", "INV"],
        [b"\n", b'"', b",", b""],
        transition=[
            [EOR, ENC, EOR, EOR, EOR, INV],      # \n
            [ENC, ESC, INV, ENC, ENC, INV],      # "
            [EOF, ENC, EOF, EOF, EOF, INV],      # ,
            [FLD, ENC, FLD, FLD, INV, INV],      # *
        ],
        emit=[
            [R, D, R, R, R, C],
            [C, C, C, C, D, C],
            [F, D, F, F, F, C],
            [D, D, D, D, C, C],
        ],
        eoi=[EOI_NONE, EOI_ERROR, EOI_RECORD, EOI_RECORD, EOI_RECORD, EOI_ERROR],
    )


def csv_comment() -> DfaTables:
    """CSV + '#' comment lines at record start (reading R19)."""
    EOR, ENC, FLD, EOF, ESC, CMT, INV = range(7)
    return DfaTables(
        "csv_comment", ["EOR", "ENC", "FLD", "EOF", "ESC", "CMT", "INV"],
        [b"\n", b'"', b",", b"#", b""],
        transition=[
            [EOR, ENC, EOR, EOR, EOR, EOR, INV],   # \n
            [ENC, ESC, INV, ENC, ENC, CMT, INV],   # "
            [EOF, ENC, EOF, EOF, EOF, CMT, INV],   # ,
            [CMT, ENC, FLD, FLD, INV, CMT, INV],   # #
            [FLD, ENC, FLD, FLD, INV, CMT, INV],   # *
        ],
        emit=[
            [R, D, R, R, R, C, C],
            [C, C, C, C, D, C, C],
            [F, D, F, F, F, C, C],
            [C, D, D, D, C, C, C],
            [D, D, D, D, C, C, C],
        ],
        eoi=[EOI_NONE, EOI_ERROR, EOI_RECORD, EOI_RECORD, EOI_RECORD, EOI_NONE, EOI_ERROR],
    )


def common_log_format() -> DfaTables:
    """Common Log Format (reading R20): 9 states, 8 groups — the "larger DFA" config."""
    EOR, FLD, EOF, QUO, QES, CLS, BRK, CMT, INV = range(9)
    return DfaTables(
        "clf", ["EOR", "FLD", "EOF", "QUO", "QES", "CLS", "BRK", "CMT", "INV"],
        [b"\n", b" ", b'"', b"[", b"]", b"\\", b"#", b""],
        transition=[
            [EOR, EOR, EOR, INV, INV, EOR, INV, EOR, INV],   # \n
            [EOF, EOF, EOF, QUO, QUO, EOF, BRK, CMT, INV],   # space
            [QUO, FLD, QUO, CLS, QUO, INV, BRK, CMT, INV],   # "
            [BRK, FLD, BRK, QUO, QUO, INV, BRK, CMT, INV],   # [
            [FLD, FLD, FLD, QUO, QUO, INV, CLS, CMT, INV],   # ]
            [FLD, FLD, FLD, QES, QUO, INV, BRK, CMT, INV],   # backslash
            [CMT, FLD, FLD, QUO, QUO, INV, BRK, CMT, INV],   # #
            [FLD, FLD, FLD, QUO, QUO, INV, BRK, CMT, INV],   # *
        ],
        emit=[
            [R, R, R, C, C, R, C, C, C],
            [F, F, F, D, D, F, D, C, C],
            [C, D, C, C, D, C, D, C, C],
            [C, D, C, D, D, C, D, C, C],
            [D, D, D, D, D, C, C, C, C],
            [D, D, D, D, D, C, D, C, C],
            [C, D, D, D, D, C, D, C, C],
            [D, D, D, D, D, C, D, C, C],
        ],
        eoi=[EOI_NONE, EOI_RECORD, EOI_RECORD, EOI_ERROR, EOI_ERROR, EOI_RECORD, EOI_ERROR, EOI_NONE,
             EOI_ERROR],
    )


DIALECTS = {"csv": rfc4180, "csv_comment": csv_comment, "clf": common_log_format}


def get(name: str) -> DfaTables:
    return DIALECTS[name]()
