"""Staleness key of a profile: the SHA-1 of one kernel's SASS in the built
library (cuobjdump -sass), so a profile is matched to the exact machine code
it measured, not to source text (comment-only edits keep the key; any code
change breaks it)."""
import hashlib
import subprocess

U32_THROUGHPUT = "_ZN4mcsg17mcs_search_kernelINS_6SearchIjLb0ENS_8WarpSmemIjLb0EEEEELb0ELb0EEEvNS_12KernelParamsE"
U64_DIRECTED_THROUGHPUT = "_ZN4mcsg17mcs_search_kernelINS_6SearchImLb1ENS_8WarpSmemImLb1EEEEELb0ELb0EEEvNS_12KernelParamsE"
U64_THROUGHPUT = "_ZN4mcsg17mcs_search_kernelINS_6SearchImLb0ENS_8WarpSmemImLb0EEEEELb0ELb0EEEvNS_12KernelParamsE"


def kernel_sass_sha1(lib_path: str, function: str):
    """SHA-1 of `function`'s SASS listing in lib_path, None when cuobjdump or
    the function is unavailable."""
    try:
        out = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True,
                             timeout=60).stdout
    except (OSError, subprocess.TimeoutExpired):
        return None
    block, on = [], False
    for line in out.splitlines():
        if "Function : " in line:
            if on:
                break
            on = line.split("Function : ", 1)[1].strip() == function
            continue
        if on:
            block.append(line)
    if not block:
        return None
    return hashlib.sha1("\n".join(block).encode()).hexdigest()


if __name__ == "__main__":
    import sys
    print(kernel_sass_sha1(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else U32_THROUGHPUT))
