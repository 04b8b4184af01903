timeout 900 python -m pytest tests -m gpu -x -q -k "units or tiny or 7b or full or rollback or exits or prefill or ar_" 2>&1 | grep -E "FAILED|Error|assert|^E " | head -30
