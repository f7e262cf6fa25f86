"""Expression tokens and host-side semantics (mirror of mbasynth.expr).

The device evaluates candidates; the host only needs the token model, the
soundness re-check of a winner (engine.py:264-269 re-verifies outside the
parallel path with ``check``, expr.py:201-218) and the infix text used in
result reports (``run_stats``, cli JSON).  Token packing is the reference's:
variable x_i -> i, operator -> -(slot + 1) in the fixed Op order
(expr.py:22-32, 66-85).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum

DEFAULT_WIDTH = 32
MAX_WIDTH = 64


class Op(IntEnum):
    """Operator slots in the fixed enumeration order (expr.py:22-32)."""

    NOT = 0
    AND = 1
    OR = 2
    XOR = 3
    NEG = 4
    ADD = 5
    SUB = 6
    MUL = 7


UNARY_OPS = (Op.NOT, Op.NEG)
BINARY_OPS = (Op.AND, Op.OR, Op.XOR, Op.ADD, Op.SUB, Op.MUL)
COMMUTATIVE_OPS = frozenset((Op.AND, Op.OR, Op.XOR, Op.ADD, Op.MUL))
_INFIX = {Op.NOT: "~", Op.AND: "&", Op.OR: "|", Op.XOR: "^", Op.NEG: "-", Op.ADD: "+", Op.SUB: "-", Op.MUL: "*"}


def op_token(op: Op) -> int:
    return -(int(op) + 1)


def var_token(index: int) -> int:
    return index


def token_op(tok: int) -> Op:
    return Op(-tok - 1)


def token_arity(tok: int) -> int:
    if tok >= 0:
        return 0
    return 1 if tok in (-1, -5) else 2


class MalformedRpnError(ValueError):
    """Token sequence is not a valid reverse Polish program."""


class InputArityError(ValueError):
    """A variable index is out of range for the supplied input tuple."""


class ParseError(ValueError):
    def __init__(self, message: str, position: int):
        super().__init__(f"at position {position}: {message}")
        self.position = position


def validate_width(w: int) -> int:
    if not 1 <= w <= MAX_WIDTH:
        raise ValueError(f"bit width must be in 1..{MAX_WIDTH}, got {w}")
    return w


@dataclass(frozen=True)
class RpnExpr:
    """A validated RPN token sequence (expr.py:114-143)."""

    tokens: tuple[int, ...]

    def __post_init__(self):
        depth = 0
        for pos, tok in enumerate(self.tokens):
            need = token_arity(tok)
            if depth < need:
                raise MalformedRpnError(f"stack underflow at token {pos} (depth {depth}, arity {need})")
            depth += 1 - need
        if depth != 1:
            raise MalformedRpnError(f"program leaves {depth} values on the stack, expected 1")

    @property
    def size(self) -> int:
        return len(self.tokens)

    def max_var_index(self) -> int:
        return max(tok for tok in self.tokens if tok >= 0)

    def __str__(self) -> str:
        return to_infix(self)


def _eval(tokens, inputs, mask: int) -> int:
    """Host RPN interpreter with the reference's semantics (expr.py:157-198)."""
    stack: list[int] = []
    for t in tokens:
        if t >= 0:
            if t >= len(inputs):
                raise InputArityError(f"variable x{t} but input has {len(inputs)} component(s)")
            stack.append(inputs[t])
            continue
        if t == -1:
            stack[-1] ^= mask
        elif t == -5:
            stack[-1] = -stack[-1] & mask
        else:
            b = stack.pop()
            a = stack[-1]
            if t == -2:
                r = a & b
            elif t == -3:
                r = a | b
            elif t == -4:
                r = a ^ b
            elif t == -6:
                r = (a + b) & mask
            elif t == -7:
                r = (a - b) & mask
            else:
                r = (a * b) & mask
            stack[-1] = r
    return stack[0]


def evaluate(expr: RpnExpr, inputs: tuple[int, ...], width: int = DEFAULT_WIDTH) -> int:
    validate_width(width)
    return _eval(expr.tokens, inputs, (1 << width) - 1)


def check(expr: RpnExpr, spec) -> bool:
    """True iff expr matches every pair of spec (expr.py:201-218)."""
    if spec.k <= expr.max_var_index():
        raise InputArityError(f"expression uses x{expr.max_var_index()} but spec has k={spec.k}")
    mask = (1 << spec.w) - 1
    for inputs, output in spec.pairs:
        if _eval(expr.tokens, inputs, mask) != output:
            return False
    return True


def observational_behavior(expr: RpnExpr, spec) -> tuple[int, ...]:
    """The outputs (e(x_1), ..., e(x_n)) in specification order (expr.py:221-229)."""
    return tuple(evaluate(expr, inputs, spec.w) for inputs, _ in spec.pairs)


def to_infix(expr: RpnExpr) -> str:
    """Fully parenthesised infix, identical text to expr.py:242-259."""
    stack: list[str] = []
    for tok in expr.tokens:
        if tok >= 0:
            stack.append(f"x{tok}")
            continue
        op = token_op(tok)
        if op in UNARY_OPS:
            child = stack.pop()
            if child.startswith("(") and child.endswith(")"):
                child = child[1:-1]
            stack.append(f"{_INFIX[op]}({child})")
        else:
            right = stack.pop()
            left = stack.pop()
            stack.append(f"({left} {_INFIX[op]} {right})")
    return stack[0]


class _Parser:
    """Recursive descent over the reference's infix grammar (expr.py:293-384):
    unary > * > +,- > &,^,| (left-associative)."""

    def __init__(self, text: str, k: int):
        self.text, self.k, self.pos = text, k, 0

    def _peek(self) -> str:
        while self.pos < len(self.text) and self.text[self.pos].isspace():
            self.pos += 1
        return self.text[self.pos] if self.pos < len(self.text) else ""

    def _level(self, ops, sub):
        toks = sub()
        while self._peek() in ops and self._peek():
            op = ops[self.text[self.pos]]
            self.pos += 1
            toks = toks + sub() + [op_token(op)]
        return toks

    def bitwise(self):
        return self._level({"&": Op.AND, "|": Op.OR, "^": Op.XOR}, self.additive)

    def additive(self):
        return self._level({"+": Op.ADD, "-": Op.SUB}, self.multiplicative)

    def multiplicative(self):
        return self._level({"*": Op.MUL}, self.unary)

    def unary(self):
        ch = self._peek()
        if ch == "~":
            self.pos += 1
            return self.unary() + [op_token(Op.NOT)]
        if ch == "-":
            self.pos += 1
            return self.unary() + [op_token(Op.NEG)]
        return self.atom()

    def atom(self):
        ch = self._peek()
        if ch == "(":
            self.pos += 1
            toks = self.bitwise()
            if self._peek() != ")":
                raise ParseError("expected ')'", self.pos)
            self.pos += 1
            return toks
        if ch == "x":
            start = self.pos
            self.pos += 1
            digits = ""
            while self.pos < len(self.text) and self.text[self.pos].isdigit():
                digits += self.text[self.pos]
                self.pos += 1
            if not digits:
                raise ParseError("expected variable index after 'x'", start)
            idx = int(digits)
            if idx >= self.k:
                raise ParseError(f"variable x{idx} out of range for k={self.k}", start)
            return [idx]
        raise ParseError("expected variable, unary operator, or '('", self.pos)

    def parse(self) -> RpnExpr:
        toks = self.bitwise()
        if self._peek():
            raise ParseError("expected end of input or binary operator", self.pos)
        return RpnExpr(tuple(toks))


def parse_infix(text: str, k: int) -> RpnExpr:
    return _Parser(text, k).parse()


def format_word(value: int, w: int) -> str:
    return f"0x{value:0{(w + 3) // 4}x}"


def parse_word(text: str, w: int) -> int:
    if not text.startswith("0x"):
        raise ValueError(f"hex word must be 0x-prefixed, got {text!r}")
    value = int(text, 16)
    if value >= 1 << w:
        raise ValueError(f"{text} does not fit in {w} bits")
    return value
